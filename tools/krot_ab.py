"""Dev tool: in-graph ImplB (default plan) over the 7B shapes and M = 1..64;
run once per FDPP_KROT setting (k-order rotation A/B)."""
import importlib
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
tag = "krot=" + os.environ.get("FDPP_KROT", "7") + " l2pd=" + os.environ.get("FDPP_L2PD", "0")
for n, k in ((12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (32000, 4096)):
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    res = []
    for m in (2, 16, 32, 64):
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        t = min(graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out) for w in ws]) / L
                for _ in range(3))
        res.append(f"M{m}:{t:6.2f}")
    print(f"{tag} [{n},{k}] " + " ".join(res), flush=True)
    del ws
