"""Dev tool: ImplC at M = 192/256 -- cluster (auto) vs persistent stream-K with
128-token tiles over 148 / 296 CTAs (balanced SM load), in-graph."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
for n, k in ((12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (11008, 4096)):
    L = max(4, min(16, int(1.2e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    for m in (192, 256):
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        res = []
        for name, kw in (("auto", {}), ("bx128-sk148", {"block_x": 128, "ctas": 148}),
                         ("bx128-sk296", {"block_x": 128, "ctas": 296}), ("bx256-sk148", {"block_x": 256, "ctas": 148})):
            try:
                t = min(graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_C, a, w, out=out, **kw) for w in ws]) / L
                        for _ in range(2))
                res.append(f"{name}:{t:6.2f}({2*m*n*k/t/1e6:5.0f}TF)")
            except Exception as e:  # noqa: BLE001
                res.append(f"{name}:ERR({str(e)[:40]})")
        print(f"[{n},{k}] M={m} " + " ".join(res), flush=True)
    del ws
