"""Dev tool: device time of ImplA/B/C over (shape, M, splits, stages)."""
import importlib
import itertools
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200.timing import measure, median_mad  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
shapes = [(12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (32000, 4096)]
Ms = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 8, 16, 32, 64]
res = []
for n, k in shapes:
    b = (torch.randn((k, n), device="cuda") / k ** 0.5).half()
    pw = fd.pack_weight(b)
    del b
    for m in Ms:
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        byt = n * k * 2 + m * k * 2 + m * n * 2
        cands = []
        if m <= 8:
            cands.append(("A", D.KernelChoice.IMPL_A, {}))
        for ct, st in itertools.product((0, 74, 296), (0, 4)):
            cands.append((f"B ct{ct} st{st}", D.KernelChoice.IMPL_B, {"ctas": ct, "stages": st}))
        cands.append(("C", D.KernelChoice.IMPL_C, {}))
        for name, ch, kw in cands:
            f = lambda: D.run_device(ch, a, pw, out=out, **kw)
            med, _ = median_mad(measure(f, reps=10, warmup=2))
            res.append({"n": n, "k": k, "m": m, "impl": name, "us": med * 1e6, "gbs": byt / med / 1e9})
            print(f"[{n},{k}] M={m:3d} {name:12s} {med*1e6:8.1f} us {byt/med/1e9:7.0f} GB/s", flush=True)
json.dump(res, open("gpurun_out/gemm_sweep.json", "w"))
