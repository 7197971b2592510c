"""Dev tool: flat GEMM (M <= 64) on CTA pairs (FDPP_PAIR_FLAT=1: one
cta_group::2 MMA per 256 weight rows, each CTA staging half the tokens) vs
ImplB; in-graph us and max row-relative error vs torch fp32."""
import importlib
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
tag = "pair" if os.environ.get("FDPP_PAIR_FLAT") else "implB"
for n, k in ((12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (32000, 4096)):
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    g = torch.Generator(device="cuda").manual_seed(n)
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda", generator=g) / k ** 0.5).half(), k, n) for _ in range(L)]
    res = []
    for m in (2, 16, 32, 64):
        a = torch.randn((m, k), device="cuda", generator=g).half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        D.run_device(D.KernelChoice.IMPL_B, a, ws[0], out=out)
        torch.cuda.synchronize()
        ref = a.float() @ ws[0].w.float().t()
        err = float(((out.float() - ref).abs().amax(1) / ref.abs().amax(1)).max())
        t = min(graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out) for w in ws]) / L
                for _ in range(3))
        res.append(f"M{m}:{t:6.2f}(e{err:.0e})")
    print(f"{tag} [{n},{k}] " + " ".join(res), flush=True)
    del ws
