"""Dev tool: flat GEMM with the weight stored as contiguous [N/128][K/64][128][64]
boxes (FDPP_WTILE=1 probe) vs the row-major [N, K] layout (unset): in-graph
time over the 7B shapes and a checksum of one output (must match across runs)."""
import importlib
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
tiled = os.environ.get("FDPP_WTILE") is not None
tag = f"wtile={int(tiled)} krot={os.environ.get('FDPP_KROT', '0')}"


def lay(w):
    n, k = w.shape
    if not tiled:
        return w
    return w.view(n // 128, 128, k // 64, 64).permute(0, 2, 1, 3).contiguous().view(n, k)


for n, k in ((12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (32000, 4096)):
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    g = torch.Generator(device="cuda").manual_seed(n + k)
    ws = [fd.PackedWeight(lay((torch.randn((n, k), device="cuda", generator=g) / k ** 0.5).half()), k, n)
          for _ in range(L)]
    res = []
    for m in (2, 16, 32, 64):
        a = torch.randn((m, k), device="cuda", generator=g).half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        D.run_device(D.KernelChoice.IMPL_B, a, ws[0], out=out)
        cks = float(out.float().abs().sum())
        t = min(graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out) for w in ws]) / L
                for _ in range(3))
        res.append(f"M{m}:{t:6.2f}({cks:.6g})")
    print(f"{tag} [{n},{k}] " + " ".join(res), flush=True)
    del ws
