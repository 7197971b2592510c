"""Dev tool: does the M-dependence of ImplB come from the activation traffic or
from the tile width?  Times (M, block_x) pairs in-graph: M=1 with a 64-wide
tile moves no extra activation bytes (TMA zero-fills rows >= M)."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
for n, k in ((12288, 4096), (4096, 4096), (4096, 11008)):
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    for m, bx in ((1, 16), (1, 32), (1, 64), (16, 16), (16, 64), (32, 32), (32, 64), (64, 64)):
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        res = []
        for st in (0, 2, 4):
            t = graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out, block_x=bx, stages=st)
                                    for w in ws]) / L
            res.append(f"st{st}={t:6.2f}us/{n*k*2/t/1e3:5.0f}")
        print(f"[{n},{k}] M={m:2d} bx={bx:2d} " + "  ".join(res), flush=True)
    del ws
