"""Dev tool: cost of each QKV-GEMM fusion (folded RMSNorm, RoPE + KV append) at M=32, in-graph."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200 import gemm  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

M, H, Hq, Hkv = 32, 4096, 32, 32
N = (Hq + 2 * Hkv) * 128
L = 16
ws = [fd.PackedWeight((torch.randn((N, H), device="cuda") / H ** 0.5).half(), H, N) for _ in range(L)]
x = torch.randn((M, H), device="cuda").half()
out = torch.empty((M, N), device="cuda").half()
ssq = torch.ones((32, M), device="cuda") * H
q = torch.empty((M, Hq, 128), device="cuda").half()
kc = torch.empty((M, Hkv, 64, 128), device="cuda").half()
vc = torch.empty_like(kc)
pos = torch.full((M,), 5, dtype=torch.int32, device="cuda")
rope = {"q_out": q, "k_cache": kc, "v_cache": vc, "pos": pos}
for name, fn in {
    "plain": lambda: [gemm.run_fused(x, w, out=out) for w in ws],
    "ssq_out": lambda: [gemm.run_fused(x, w, out=out, ssq_out=torch.empty(0)) for w in ws][:0] or
                       [gemm.run_fused(x, w, out=out) for w in ws],
    "x_op3": lambda: [gemm.run_fused(x, w, out=out, x_op=3, ssq_in=ssq, ssq_tiles=32) for w in ws],
    "rope": lambda: [gemm.run_fused(x, w, rope=rope) for w in ws],
    "x_op3+rope": lambda: [gemm.run_fused(x, w, x_op=3, ssq_in=ssq, ssq_tiles=32, rope=rope) for w in ws],
}.items():
    t = graph_time(fn) / L
    print(f"{name:12s} {t:6.2f} us  {N * H * 2 / t / 1e3:5.0f} GB/s", flush=True)
