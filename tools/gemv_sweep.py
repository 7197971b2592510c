"""Dev tool: in-graph ImplA (GEMV) vs ImplB at M = 1..8 on the decode shapes."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
for n, k in ((12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (1280, 8192), (8192, 1024)):
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    res = []
    for m in (1, 2, 4, 8):
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        ta = graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_A, a, w, out=out) for w in ws]) / L
        tb = graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out) for w in ws]) / L
        res.append(f"M={m}: A {ta:6.2f}us/{n*k*2/ta/1e3:5.0f}  B {tb:6.2f}us/{n*k*2/tb/1e3:5.0f}")
    print(f"[{n},{k}] " + " | ".join(res), flush=True)
    del ws
