"""Dev tool for ncu: isolate fixed per-launch costs of the tcgen05 GEMM."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
cases = [  # (n, k, m, ctas, stages)
    (4096, 64, 32, 0, 0), (4096, 64, 32, 32, 0), (4096, 64, 32, 32, 1),
    (128, 64, 32, 1, 1), (4096, 4096, 32, 0, 0), (4096, 4096, 32, 0, 4), (4096, 4096, 32, 32, 0),
]
for n, k, m, ctas, st in cases:
    b = (torch.randn((k, n), device="cuda") / k ** 0.5).half()
    pw = fd.pack_weight(b)
    a = torch.randn((m, k), device="cuda").half()
    out = torch.empty((m, n), device="cuda", dtype=torch.half)
    for i in range(3):
        D.run_device(D.KernelChoice.IMPL_B, a, pw, out=out, ctas=ctas, stages=st)
    torch.cuda.synchronize()
    print("case", n, k, m, ctas, st, flush=True)
