"""Dev tool: what the QKV projection's fused epilogue costs, in-graph at M = 1..64
on [12288, 4096]: plain ImplB, + folded RMSNorm (x_op 3), + RoPE/KV append."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200 import gemm  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

n, k, Hq, Hkv, Lc = 12288, 4096, 32, 32, 1100
L = 12
ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
for m in (1, 8, 32, 64):
    x = torch.randn((m, k), device="cuda").half()
    out = torch.empty((m, n), device="cuda", dtype=torch.half)
    ssq = (x.float() ** 2).sum(1).view(1, m).contiguous()
    q = torch.empty((m, Hq, 128), device="cuda", dtype=torch.half)
    kc = torch.zeros((m, Hkv, Lc, 128), device="cuda", dtype=torch.half)
    vc = torch.zeros_like(kc)
    pos = torch.full((m,), 1024, device="cuda", dtype=torch.int32)
    rope = {"q_out": q, "k_cache": kc, "v_cache": vc, "pos": pos, "theta": 10000.0}
    variants = {
        "plain": lambda w: gemm.run_fused(x, w, out=out),
        "rmsnorm": lambda w: gemm.run_fused(x, w, out=out, x_op=3, ssq_in=ssq, ssq_tiles=1),
        "rope": lambda w: gemm.run_fused(x, w, rope=rope),
        "rmsnorm+rope": lambda w: gemm.run_fused(x, w, x_op=3, ssq_in=ssq, ssq_tiles=1, rope=rope),
    }
    res = []
    for name, f in variants.items():
        t = min(graph_time(lambda: [f(w) for w in ws]) / L for _ in range(3))
        res.append(f"{name}:{t:6.2f}")
    print(f"[{n},{k}] M={m:2d} " + " ".join(res), flush=True)
