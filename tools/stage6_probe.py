"""Dev tool: ImplB at M <= 16 (16-token tiles) with the default 5-stage ring vs 6 stages
(109 KB: two CTAs still fit an SM), in-graph over rotating weights."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
for n, k in ((12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (32000, 4096)):
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    res = []
    for m in (1, 8, 16):
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        for s in (0, 6):
            t = min(graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out, stages=s) for w in ws]) / L
                    for _ in range(3))
            res.append(f"M{m}/s{s or 5}:{t:6.2f}")
    print(f"[{n},{k}] " + " ".join(res), flush=True)
    del ws
