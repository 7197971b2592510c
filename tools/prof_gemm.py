"""Dev tool for ncu: run one GEMM impl a few times (no timing, no flush)."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
n, k, m = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
impl = {"A": D.KernelChoice.IMPL_A, "B": D.KernelChoice.IMPL_B, "C": D.KernelChoice.IMPL_C}[sys.argv[4]]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
ws = []
for i in range(4):  # rotate 4 weight copies so consecutive launches miss L2
    b = (torch.randn((k, n), device="cuda") / k ** 0.5).half()
    ws.append(fd.pack_weight(b))
a = torch.randn((m, k), device="cuda").half()
out = torch.empty((m, n), device="cuda", dtype=torch.half)
for i in range(reps):
    D.run_device(impl, a, ws[i % 4], out=out)
torch.cuda.synchronize()
print("done")
