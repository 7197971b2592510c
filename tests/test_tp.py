"""Tensor-parallel decode layer on CPU: the shard
mapping of tp.py plus one all-reduce after O and after down (rank 0 adds the
residual) must reproduce the unsharded layer.  world_size 2 and 4 over gloo,
fp32 torch restatement (tp.reference_layer) -- the same shard functions the
CUDA LlamaDecoder uses on the GPU."""

import math
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2311_01282_b200 import tp  # noqa: E402
from paper_2311_01282_b200.llama import LLAMA2_70B, LlamaConfig  # noqa: E402

TINY = LlamaConfig("tiny-gqa", hidden=128, n_heads=8, n_kv_heads=4, head_dim=16, ffn=192,
                   n_layers=2, vocab=64)


def _model(cfg, seed=0):
    g = torch.Generator().manual_seed(seed)

    def w(n, k):
        return torch.randn((n, k), generator=g) / math.sqrt(k)

    D = cfg.head_dim
    layers = [{"qkv": w((cfg.n_heads + 2 * cfg.n_kv_heads) * D, cfg.hidden),
               "o": w(cfg.hidden, cfg.n_heads * D), "gate_up": w(2 * cfg.ffn, cfg.hidden),
               "down": w(cfg.hidden, cfg.ffn),
               "ln1": 1 + 0.1 * torch.randn(cfg.hidden, generator=g),
               "ln2": 1 + 0.1 * torch.randn(cfg.hidden, generator=g)} for _ in range(cfg.n_layers)]
    B, Lmax = 3, 40
    kc = [torch.randn((B, cfg.n_kv_heads, Lmax, D), generator=g) for _ in range(cfg.n_layers)]
    vc = [torch.randn((B, cfg.n_kv_heads, Lmax, D), generator=g) for _ in range(cfg.n_layers)]
    x = torch.randn((B, cfg.hidden), generator=g)
    pos = torch.tensor([5, 17, 33])
    return layers, kc, vc, x, pos


def _full_step(cfg):
    layers, kc, vc, x, pos = _model(cfg)
    for li, L in enumerate(layers):
        x = tp.reference_layer(x, L, kc[li], vc[li], pos, pos + 1, cfg, cfg.n_heads, cfg.n_kv_heads)
    return x, kc, vc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = TINY
        layers, kc, vc, x, pos = _model(cfg)
        s = tp.shard_dims(cfg, world)
        for li, L in enumerate(layers):
            Ls = tp.shard_layer(L, cfg, rank, world)
            kcs, vcs = tp.shard_cache(kc[li], cfg, rank, world), tp.shard_cache(vc[li], cfg, rank, world)
            x = tp.reference_layer(x, Ls, kcs, vcs, pos, pos + 1, cfg, s.n_heads, s.n_kv_heads,
                                   rank=rank, all_reduce=dist.all_reduce)
            kc[li][:, rank * s.n_kv_heads:(rank + 1) * s.n_kv_heads] = kcs
            vc[li][:, rank * s.n_kv_heads:(rank + 1) * s.n_kv_heads] = vcs
        # numpy copies travel by value: a shared-memory tensor would need the
        # worker alive until the parent has unpickled it
        q.put((rank, x.numpy().copy(),
               [k[:, rank * s.n_kv_heads:(rank + 1) * s.n_kv_heads].numpy().copy() for k in kc]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_tp_layer_matches_unsharded(world):
    ref_x, ref_kc, _ = _full_step(TINY)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = tp.shard_dims(TINY, world)
    for rank, x, kcs in got:
        x, kcs = torch.from_numpy(x), [torch.from_numpy(k) for k in kcs]
        assert torch.allclose(x, ref_x, atol=2e-4, rtol=2e-4), f"rank {rank}: residual stream differs"
        for li in range(TINY.n_layers):  # each rank appended its own KV heads' rows
            exp = ref_kc[li][:, rank * s.n_kv_heads:(rank + 1) * s.n_kv_heads]
            assert torch.allclose(kcs[li], exp, atol=1e-5)


def test_shard_shapes_70b():
    # t = 2/4/8 -> 4/2/1 KV heads and 32/16/8 query heads per GPU (G = 8)
    for t, kv, q in ((2, 4, 32), (4, 2, 16), (8, 1, 8)):
        s = tp.shard_dims(LLAMA2_70B, t)
        assert (s.n_kv_heads, s.n_heads, s.ffn) == (kv, q, 28672 // t)
        sh = tp.rank_gemm_shapes(LLAMA2_70B, t)
        assert sh["qkv"] == ((q + 2 * kv) * 128, 8192)
        assert sh["o"] == (8192, q * 128) and sh["down"] == (8192, 28672 // t)
        assert sh["gate_up"] == (2 * 28672 // t, 8192)


def test_shard_partition_is_exact():
    # concatenating every rank's shard recovers the full weight (no row lost / duplicated)
    layers, *_ = _model(TINY)
    L = layers[0]
    t = 4
    D, Hq, Hkv, f = TINY.head_dim, TINY.n_heads, TINY.n_kv_heads, TINY.ffn
    shards = [tp.shard_layer(L, TINY, r, t) for r in range(t)]
    o = torch.cat([s["o"] for s in shards], 1)
    assert torch.equal(o, L["o"])
    assert torch.equal(torch.cat([s["down"] for s in shards], 1), L["down"])
    qs = torch.cat([s["qkv"][:Hq // t * D] for s in shards], 0)
    assert torch.equal(qs, L["qkv"][:Hq * D])
    gates = torch.cat([s["gate_up"][:f // t] for s in shards], 0)
    ups = torch.cat([s["gate_up"][f // t:] for s in shards], 0)
    assert torch.equal(gates, L["gate_up"][:f]) and torch.equal(ups, L["gate_up"][f:])


def test_shard_errors():
    with pytest.raises(ValueError):
        tp.shard_dims(TINY, 3)
    with pytest.raises(ValueError):
        tp.shard_dims(TINY, 0)
