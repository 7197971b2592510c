"""The one-shot all-reduce fused into the row-parallel GEMM epilogue
(allreduce.py, fdpp_gemm_fuse.ar_*).

This pod has one GPU, so the exchange is exercised with several "ranks" in
one process on cuda:0, each rank's kernel on its own stream with its own
workspace (the peer pointers are plain device pointers instead of CUDA IPC
mappings; the kernel code is the same).  The multi-GPU form (IPC-mapped
workspaces, one process per GPU) runs when two GPUs are visible."""

import math
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


def _run_ranks(torch, ars, fn):
    """Launch fn(rank) for every rank on its own stream (concurrently)."""
    streams = [torch.cuda.Stream() for _ in ars]
    torch.cuda.synchronize()
    for r, s in enumerate(streams):
        with torch.cuda.stream(s):
            fn(r)
    torch.cuda.synchronize()
    for ar in ars:
        assert not ar.timed_out(), "a rank timed out waiting for its peers"


@pytest.mark.parametrize("world", [2, 4])
def test_fused_allreduce_gemm(torch, world):
    """C = x + sum_r A_r W_r^T with ssq_out, over `world` ranks, for alternating
    call sites (O-like K = 512 and down-like K = 1536, M = 8 / 32): every rank's
    C is bitwise identical (same rank-order sum), within the fp16 bar of the
    fp32 reference; epochs and the two receive parities cycle correctly."""
    from paper_2311_01282_b200 import gemm
    from paper_2311_01282_b200.allreduce import PeerAllReduce
    N = 1024
    ars = PeerAllReduce.local_group(world, cap=64 * N)
    g = torch.Generator(device="cuda").manual_seed(world)
    try:
        for call, (M, K) in enumerate([(8, 512), (32, 1536), (8, 512), (32, 1536), (16, 512)]):
            A = [torch.randn((M, K), generator=g, device="cuda").half() for _ in range(world)]
            W = [gemm.PackedWeight((torch.randn((N, K), generator=g, device="cuda") / math.sqrt(K * world)).half(),
                                   K, N) for _ in range(world)]
            x = torch.randn((M, N), generator=g, device="cuda").half()
            xs = [x.clone() for _ in range(world)]
            ssq = [torch.zeros((N // 128, M), device="cuda") for _ in range(world)]

            def step(r):
                gemm.run_fused(A[r], W[r], out=xs[r], residual=xs[r], ssq_out=ssq[r], allreduce=ars[r],
                               ws_tag=f"ar{r}")
            _run_ranks(torch, ars, step)
            ref = x.float() + sum(A[r].float() @ W[r].w.float().t() for r in range(world))
            for r in range(1, world):
                assert torch.equal(xs[r], xs[0]), f"call {call}: rank {r} differs from rank 0"
            err = ((xs[0].float() - ref).abs().amax(1) / ref.abs().amax(1)).max().item()
            assert err <= 2e-3, f"call {call}: rel err {err}"
            ssq_ref = (xs[0].float() ** 2).view(M, N // 128, 128).sum(-1).t()
            assert torch.allclose(ssq[0], ssq_ref, rtol=1e-4, atol=1e-3)
    finally:
        for ar in ars:
            ar.close()


def test_fused_allreduce_decode_step(torch):
    """Two tensor-parallel ranks of the decode step with the all-reduce fused
    into the O / down epilogues (residual and next-RMSNorm sums of squares in
    the same epilogue): equals the unsharded decoder's step."""
    import importlib
    from paper_2311_01282_b200 import llama, tp
    from paper_2311_01282_b200.allreduce import PeerAllReduce
    from tests.test_gpu_tp import _setup, _state, _table
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

    world = 2
    ars = PeerAllReduce.local_group(world, cap=4 * cfg.hidden)
    try:
        decs = []
        for r in range(world):
            d = llama.LlamaDecoder(cfg, 4, 72, table=_table(D, cfg, world), weights=W, tp_rank=r, tp_size=world,
                                   allreduce=ars[r])
            for li in range(cfg.n_layers):
                d.k_cache[li].copy_(tp.shard_cache(kc[li], cfg, r, world))
                d.v_cache[li].copy_(tp.shard_cache(vc[li], cfg, r, world))
            d.ids.copy_(ids)
            d.pos.copy_(pos)
            d.lens.copy_(pos + 1)
            decs.append(d)
        _run_ranks(torch, ars, lambda r: decs[r].enqueue_step())
        for r, d in enumerate(decs):
            x = d.x.float().cpu().numpy()
            err = float((np.abs(x - x_ref).max(1) / np.abs(x_ref).max(1)).max())
            assert err <= 2e-2, f"rank {r}: rel err {err}"
        assert torch.equal(decs[0].x, decs[1].x)
        assert torch.equal(decs[0].ids, decs[1].ids)
    finally:
        for ar in ars:
            ar.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mgpu_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2311_01282_b200 import gemm
        from paper_2311_01282_b200.allreduce import PeerAllReduce
        ar = PeerAllReduce.create(dist.group.WORLD, cap=32 * 4096)
        g = torch.Generator(device="cuda").manual_seed(rank)
        M, K, N = 32, 1024, 4096
        a = torch.randn((M, K), generator=g, device="cuda").half()
        w = gemm.PackedWeight((torch.randn((N, K), generator=g, device="cuda") / 64).half(), K, N)
        x = torch.ones((M, N), device="cuda").half()
        dist.barrier()
        gemm.run_fused(a, w, out=x, residual=x, allreduce=ar)
        part = (a.float() @ w.w.float().t())
        dist.all_reduce(part)
        torch.cuda.synchronize()
        err = ((x.float() - (part + 1)).abs().amax(1) / (part + 1).abs().amax(1)).max().item()
        q.put((rank, err, ar.timed_out()))
        dist.barrier()
        ar.close()
    finally:
        dist.destroy_process_group()


def test_fused_allreduce_two_gpus(torch):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (IPC-mapped peer workspaces over NVLink)")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mgpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, err, to in got:
        assert not to and err <= 2e-3, (rank, err, to)
