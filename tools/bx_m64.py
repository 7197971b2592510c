"""Dev tool: ImplB at M = 48/64 with one 64-token tile vs two 32-token tiles
(block_x = 32: the weight tile is read by two CTAs, the second mostly from L2)."""
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
    for m in (48, 64):
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        ref = None
        res = []
        for bx in (0, 32, 16):
            try:
                D.run_device(D.KernelChoice.IMPL_B, a, ws[0], out=out, block_x=bx)
                o = out.float().clone()
                ref = o if ref is None else ref
                err = float((o - ref).abs().max())
                t = min(graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out, block_x=bx)
                                            for w in ws]) / L for _ in range(3))
                res.append(f"bx{bx}:{t:6.2f}(d{err:.1e})")
            except Exception as e:  # noqa: BLE001
                res.append(f"bx{bx}:ERR({str(e)[:50]})")
        print(f"[{n},{k}] M={m} " + " ".join(res), flush=True)
    del ws
