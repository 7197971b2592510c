"""Dev tool: ImplB vs ImplC (cluster split-K and persistent stream-K) across
the conventional-GEMM regime M = 64..256 on the Llama-2-7B shapes, in-graph
with rotating weights (> L2), like bench.py's configs[1] sweep.

    python tools/conv_sweep.py [M,M,...]  -> gpurun_out/conv_sweep.json
"""
import importlib
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2311_01282_b200 as fd  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
peak, _ = bench._peaks()
Ms = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [32, 64, 96, 128, 192, 256]
only_m = os.environ.get("CONV_SWEEP_M")
res = []
for n, k in ((12288, 4096), (4096, 4096), (11008, 4096), (4096, 11008), (22016, 4096)):
    nrot = max(4, min(16, int(1.2e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(nrot)]
    for m in Ms:
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        byt = n * k * 2 + m * k * 2 + m * n * 2
        for name, ch, kw in (("B", D.KernelChoice.IMPL_B, {}), ("C", D.KernelChoice.IMPL_C, {}),
                             ("C-streamK", D.KernelChoice.IMPL_C, {"ctas": 148}),
                             ("C-bx128", D.KernelChoice.IMPL_C, {"block_x": 128}),
                             ("C-bx128-cs2", D.KernelChoice.IMPL_C, {"block_x": 128, "ctas": -2})):
            if name.startswith("C-bx128") and m <= 128:
                continue
            t = bench._rotating_graph_time(torch, [lambda w=w: D.run_device(ch, a, w, out=out, **kw) for w in ws])
            r = {"n": n, "k": k, "m": m, "impl": name, "us": round(t * 1e6, 2),
                 "gbs": round(byt / t / 1e9, 1), "frac": round(byt / t / 1e9 / peak, 3)}
            res.append(r)
            print(json.dumps(r), flush=True)
    del ws
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "conv_sweep.json"), "w"))
