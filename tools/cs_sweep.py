"""Dev tool: in-graph ImplB time vs cluster split-K size cs (ctas = -cs) and stream-K grids."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
Ms = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 32, 64]
cases = {(12288, 4096): (-2, -3, -4, -5, -6), (4096, 4096): (-4, -6, -8, -9, -10, -12, -16),
         (4096, 11008): (-4, -6, -8, -9, -10, -12, -16), (22016, 4096): (-1, -2, 148, 296),
         (32000, 4096): (-1, -2, 148, 296)}
for (n, k), modes in cases.items():
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    for m in Ms:
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        res = []
        for c in (0,) + modes:
            try:
                t = graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out, ctas=c) for w in ws]) / L
                res.append(f"{c}:{t:6.2f}/{n*k*2/t/1e3:4.0f}")
            except Exception as e:  # noqa: BLE001
                res.append(f"{c}:ERR({str(e)[:40]})")
        print(f"[{n},{k}] M={m:2d} " + " ".join(res), flush=True)
    del ws
