"""Dev tool: in-graph ImplB time vs ring depth (stages = 2 / 4 / default) at
M = 16 / 32 / 64: how sensitive the flat GEMM is to weight bytes in flight."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
for n, k in ((12288, 4096), (4096, 11008), (22016, 4096), (4096, 4096)):
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    for m in (16, 32, 64):
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        res = []
        for bx in (0, 32) if m <= 32 else (0,):
            for s in (1, 2, 4, 0):
                t = graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out, stages=s, block_x=bx)
                                        for w in ws]) / L
                res.append(f"bx{bx}/s{s}:{t:6.2f}")
        print(f"[{n},{k}] M={m:2d} " + " ".join(res), flush=True)
    del ws
