"""Dev tool: flat GEMM / GEMV time vs the packed weight's row pitch (ldw = K +
pad elements): does breaking the power-of-two row stride help the DRAM/L2
access pattern of the 128-row x 128-B TMA boxes?"""
import importlib
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
for n, k in ((12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (32000, 4096)):
    L = max(4, min(16, int(1.6e9 // (n * k * 2))))
    for pad in (0, 8, 64, 128, 0):
        ws = []
        for _ in range(L):
            base = torch.empty((n, k + pad), device="cuda", dtype=torch.half)
            base[:, :k] = (torch.randn((n, k), device="cuda") / k ** 0.5).half()
            ws.append(fd.PackedWeight(base[:, :k] if pad else base, k, n))
        res = []
        for m, ch in ((1, D.KernelChoice.IMPL_A), (2, D.KernelChoice.IMPL_B), (32, D.KernelChoice.IMPL_B),
                      (64, D.KernelChoice.IMPL_B)):
            a = torch.zeros((m, k + pad), device="cuda").half()
            a[:, :k] = torch.randn((m, k), device="cuda").half()
            out = torch.empty((m, n), device="cuda", dtype=torch.half)
            t = min(graph_time(lambda: [D.run_device(ch, a, w, out=out) for w in ws]) / L for _ in range(3))
            res.append(f"M{m}:{t:6.2f}")
        print(f"[{n},{k}] pad={pad:3d} " + " ".join(res), flush=True)
        del ws
