"""Dev tool for ncu: one launch of each flat-GEMM kernel kind on a Llama-2-7B
shape ([12288, 4096]): ImplA GEMV at M=4, ImplB cluster split-K at M=32,
ImplB stream-K at [22016..] M=32 forced, ImplC at M=64."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
n, k = 12288, 4096
ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(3)]
for m, ch, ctas in ((4, D.KernelChoice.IMPL_A, 0), (32, D.KernelChoice.IMPL_B, 0),
                    (32, D.KernelChoice.IMPL_B, 296), (64, D.KernelChoice.IMPL_C, 0)):
    a = torch.randn((m, k), device="cuda").half()
    for w in ws:
        D.run_device(ch, a, w, ctas=ctas)
torch.cuda.synchronize()
print("done")
