"""Dev tool: in-graph ImplB time for every cluster split cs with tiles * cs <= 2 * 148
(balanced k-ranges), on the shapes whose power-of-two auto split leaves SMs idle."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
shapes = [(4608, 4096), (10240, 8192), (5120, 8192), (2560, 8192), (1280, 8192), (12288, 4096), (4096, 4096),
          (8192, 8192), (7168, 8192)]
for n, k in shapes:
    tiles = (n + 127) // 128
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    for m in (8, 32):
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        res = []
        for c in [0] + [-c for c in range(1, 17) if tiles * c <= 296]:
            t = min(graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out, ctas=c) for w in ws]) / L
                    for _ in range(2))
            res.append(f"{-c if c else 'auto'}:{t:.2f}")
        print(f"[{n},{k}] tiles={tiles} M={m} " + " ".join(res), flush=True)
    del ws
