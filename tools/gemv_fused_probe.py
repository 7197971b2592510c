"""Dev tool: fused GEMV (fdpp_gemv_fused) variants vs the plain GEMV at M=1, in-graph."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200 import gemm  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
for n, k in ((12288, 4096), (22016, 4096)):
    L = 12
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    a = torch.randn((1, k), device="cuda").half()
    out = torch.empty((1, n), device="cuda", dtype=torch.half)
    ssq = torch.ones((512, 1), device="cuda")
    act = torch.empty((1, n // 2), device="cuda", dtype=torch.half)
    variants = {
        "plain": lambda: [D.run_device(D.KernelChoice.IMPL_A, a, w, out=out) for w in ws],
        "fused x_op0": lambda: [gemm.run_fused(a, w, out=out, impl="A") for w in ws],
        "fused x_op3(1 tile)": lambda: [gemm.run_fused(a, w, out=out, x_op=3, ssq_in=ssq, ssq_tiles=1, impl="A") for w in ws],
        "fused x_op3(512)": lambda: [gemm.run_fused(a, w, out=out, x_op=3, ssq_in=ssq, ssq_tiles=512, impl="A") for w in ws],
        "fused silu": lambda: [gemm.run_fused(a, w, silu_out=act, impl="A") for w in ws],
    }
    res = []
    for name, fn in variants.items():
        t = graph_time(fn) / L
        res.append(f"{name}: {t:6.2f}us/{n*k*2/t/1e3:5.0f}")
    print(f"[{n},{k}] " + " | ".join(res), flush=True)
    del ws
