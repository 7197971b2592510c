"""Dev tool: the CTA-pair ImplC (FDPP_IMPLC_PAIR=1) -- correctness vs a torch
fp32 reference, then in-graph time against the one-CTA plan at M = 192 / 256."""
import importlib
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
tag = {"1": "pair", "0": "one-CTA"}.get(os.environ.get("FDPP_IMPLC_PAIR"), "auto")
for n, k in ((1408, 1024), (12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (11008, 4096), (32000, 4096), (8192, 8192), (4608, 4096), (10240, 8192), (57344, 8192)):
    L = max(4, min(16, int(1.2e9 // (n * k * 2))))
    g = torch.Generator(device="cuda").manual_seed(n)
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda", generator=g) / k ** 0.5).half(), k, n) for _ in range(L)]
    res = []
    for m in (129, 192, 256):
        a = torch.randn((m, k), device="cuda", generator=g).half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        D.run_device(D.KernelChoice.IMPL_C, a, ws[0], out=out)
        torch.cuda.synchronize()
        ref = a.float() @ ws[0].w.float().t()
        err = float(((out.float() - ref).abs().amax(1) / ref.abs().amax(1)).max())
        t = min(graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_C, a, w, out=out) for w in ws]) / L
                for _ in range(2))
        res.append(f"M{m}:{t:6.2f}us {2*m*n*k/t/1e6:4.0f}TF err={err:.1e}")
    print(f"{tag} [{n},{k}] " + " ".join(res), flush=True)
    del ws
