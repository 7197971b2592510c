"""Tensor-parallel decode step through the CUDA kernels: two
ranks share cuda:0 (this pod has one GPU), each runs its LlamaDecoder shard
(sharded QKV / gate|up / O / down, local KV heads, rank 0 adds the residual in
the row-parallel epilogues, fdpp_row_ssq after each all-reduce) with a gloo
all-reduce of the residual stream; the result must equal the unsharded
decoder's step on the same weights, KV state and tokens."""

import math
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(seed=0):
    import torch
    from paper_2311_01282_b200 import llama
    cfg = llama.LlamaConfig("tiny-gqa", hidden=1024, n_heads=8, n_kv_heads=2, head_dim=128, ffn=1536,
                            n_layers=2, vocab=512)
    g = torch.Generator().manual_seed(seed)

    def w(n, k):
        return torch.randn((n, k), generator=g) / math.sqrt(k)

    D = cfg.head_dim
    W = {"layers": [{"qkv": w((cfg.n_heads + 2 * cfg.n_kv_heads) * D, cfg.hidden),
                     "o": w(cfg.hidden, cfg.n_heads * D), "gate_up": w(2 * cfg.ffn, cfg.hidden),
                     "down": w(cfg.hidden, cfg.ffn),
                     "ln1": 1 + 0.1 * torch.randn(cfg.hidden, generator=g),
                     "ln2": 1 + 0.1 * torch.randn(cfg.hidden, generator=g)} for _ in range(cfg.n_layers)],
         "embed": torch.randn((cfg.vocab, cfg.hidden), generator=g),
         "lm_head": w(cfg.vocab, cfg.hidden), "ln_f": 1 + 0.1 * torch.randn(cfg.hidden, generator=g)}
    return cfg, W


def _table(D, cfg, tp):
    t = D.DispatchTable(fingerprint="test")
    for n, k in cfg.gemm_shapes(tp).values():
        t.add(D.DispatchEntry(n=n, k=k, m1=1, m2=128))
    return t


def _worker(rank, world, port, q):
    import importlib

    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_01282_b200 import llama, tp
        D = importlib.import_module("paper_2311_01282_b200.dispatch")
        cfg, W = _setup()
        dec = llama.LlamaDecoder(cfg, 4, 72, table=_table(D, cfg, world), weights=W, tp_rank=rank,
                                 tp_size=world, group=dist.group.WORLD)
        # the same synthetic state as the unsharded decoder: full caches, then this rank's heads
        full_k, full_v, ids, pos = _state(torch, cfg)
        for li in range(cfg.n_layers):
            dec.k_cache[li].copy_(tp.shard_cache(full_k[li], cfg, rank, world))
            dec.v_cache[li].copy_(tp.shard_cache(full_v[li], cfg, rank, world))
        dec.ids.copy_(ids)
        dec.pos.copy_(pos)
        dec.lens.copy_(pos + 1)
        dec.enqueue_step()      # eager: the gloo all-reduce is not graph-capturable
        torch.cuda.synchronize()
        q.put((rank, dec.x.float().cpu().numpy(), dec.ids.cpu().numpy()))  # by value
    finally:
        dist.destroy_process_group()


def _state(torch, cfg, B=4, L=64):
    g = torch.Generator().manual_seed(7)
    kc = [torch.randn((B, cfg.n_kv_heads, 72, cfg.head_dim), generator=g).half().cuda() for _ in range(cfg.n_layers)]
    vc = [torch.randn((B, cfg.n_kv_heads, 72, cfg.head_dim), generator=g).half().cuda() for _ in range(cfg.n_layers)]
    ids = torch.randint(0, cfg.vocab, (B,), generator=g, dtype=torch.int32).cuda()
    pos = torch.full((B,), L, dtype=torch.int32).cuda()
    return kc, vc, ids, pos


def test_tp2_step_matches_unsharded():
    import importlib

    import numpy as np
    import torch
    import torch.multiprocessing as mp
    from paper_2311_01282_b200 import llama
    D = importlib.import_module("paper_2311_01282_b200.dispatch")
    cfg, W = _setup()
    ref = llama.LlamaDecoder(cfg, 4, 72, table=_table(D, cfg, 1), weights=W)
    kc, vc, ids, pos = _state(torch, cfg)
    for li in range(cfg.n_layers):
        ref.k_cache[li].copy_(kc[li])
        ref.v_cache[li].copy_(vc[li])
    ref.ids.copy_(ids)
    ref.pos.copy_(pos)
    ref.lens.copy_(pos + 1)
    ref.enqueue_step()
    torch.cuda.synchronize()
    x_ref = ref.x.float().cpu()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, x, nxt in got:
        err = float((np.abs(x - x_ref.numpy()).max(1) / np.abs(x_ref.numpy()).max(1)).max())
        assert err <= 2e-2, f"rank {rank}: rel err {err}"
    # the replicated LM head + argmax agree across ranks
    assert np.array_equal(got[0][2], got[1][2])


def _nccl_worker(rank, world, port, q):
    import importlib

    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2311_01282_b200 import llama, tp
        D = importlib.import_module("paper_2311_01282_b200.dispatch")
        cfg, W = _setup()
        dec = llama.LlamaDecoder(cfg, 4, 72, table=_table(D, cfg, world), weights=W, tp_rank=rank,
                                 tp_size=world, group=dist.group.WORLD)
        full_k, full_v, ids, pos = _state(torch, cfg)
        for li in range(cfg.n_layers):
            dec.k_cache[li].copy_(tp.shard_cache(full_k[li].to(f"cuda:{rank}"), cfg, rank, world))
            dec.v_cache[li].copy_(tp.shard_cache(full_v[li].to(f"cuda:{rank}"), cfg, rank, world))
        dec.ids.copy_(ids)
        dec.pos.copy_(pos)
        dec.lens.copy_(pos + 1)
        dec.capture()          # NCCL all-reduces inside the step's CUDA graph
        dec.step()
        torch.cuda.synchronize()
        q.put((rank, dec.x.float().cpu().numpy(), dec.ids.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_tp2_nccl_step_matches_unsharded():
    """Two GPUs, one rank each, NCCL all-reduces captured in the CUDA graph:
    the tensor-parallel step equals the unsharded decoder's (skipped on a
    single-GPU box)."""
    import importlib

    import numpy as np
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_2311_01282_b200 import llama
    D = importlib.import_module("paper_2311_01282_b200.dispatch")
    cfg, W = _setup()
    ref = llama.LlamaDecoder(cfg, 4, 72, table=_table(D, cfg, 1), weights=W)
    kc, vc, ids, pos = _state(torch, cfg)
    for li in range(cfg.n_layers):
        ref.k_cache[li].copy_(kc[li])
        ref.v_cache[li].copy_(vc[li])
    ref.ids.copy_(ids)
    ref.pos.copy_(pos)
    ref.lens.copy_(pos + 1)
    ref.enqueue_step()
    torch.cuda.synchronize()
    x_ref = ref.x.float().cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, x, nxt in got:
        err = float((np.abs(x - x_ref).max(1) / np.abs(x_ref).max(1)).max())
        assert err <= 2e-2, f"rank {rank}: rel err {err}"
    assert np.array_equal(got[0][2], got[1][2])
