"""Dev tool: in-graph per-launch time of auto ImplB per decode shape (one line per shape)."""
import importlib
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402
sys.path.insert(0, "tools")
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
Ms = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 32, 64]
tag = os.environ.get("FDPP_L2PF", "0")
for n, k in ((12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008)):
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    res = []
    for m in Ms:
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        t = graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out) for w in ws]) / L
        res.append(f"M={m}:{t:6.2f}us/{n*k*2/t/1e3:5.0f}")
    print(f"pf={tag} [{n},{k}] " + "  ".join(res), flush=True)
    del ws
