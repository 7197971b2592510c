"""Dev tool: cluster residency (cudaOccupancyMaxActiveClusters, printed by the
library under FDPP_OCC_PROBE=1) and in-graph ImplB time vs cluster split size,
including non-power-of-two splits (balanced k-ranges); plus the residency of the
attention's cluster plans."""
import math
import os
import sys

os.environ.setdefault("FDPP_OCC_PROBE", "1")
import torch  # noqa: E402

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import importlib  # noqa: E402

import paper_2311_01282_b200 as fd  # noqa: E402
from mode_sweep_lib import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
Ms = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 32, 64]
cases = {(4096, 4096): (-4, -5, -6, -7, -8, -9), (4096, 11008): (-5, -6, -7, -8, -9),
         (12288, 4096): (-1, -2, -3), (8192, 3584): (-2, -3, -4, -5), (1280, 8192): (-8, -12, -14, -16)}
for (n, k), modes in cases.items():
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    for m in Ms:
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        res = []
        for c in (0,) + modes:
            try:
                print(f"-- [{n},{k}] M={m} ctas={c}", file=sys.stderr, flush=True)
                D.run_device(D.KernelChoice.IMPL_B, a, ws[0], out=out, ctas=c)
                torch.cuda.synchronize()
                t = graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, a, w, out=out, ctas=c) for w in ws]) / L
                res.append(f"{c}:{t:6.2f}/{n*k*2/t/1e3:4.0f}")
            except Exception as e:  # noqa: BLE001
                res.append(f"{c}:ERR({str(e)[:40]})")
        print(f"[{n},{k}] M={m:2d} " + " ".join(res), flush=True)
    del ws

cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
for B, Hq, Hkv, Ln in ((8, 32, 2, 32768), (32, 32, 32, 1024), (1, 32, 32, 1024), (32, 8, 1, 1024)):
    kk = torch.randn((B, Hkv, Ln, 128), device="cuda").half()
    q = torch.randn((B, Hq, 128), device="cuda").half()
    cfg = fd.AttentionConfig(p="auto", scale=1 / math.sqrt(128), calib=cal)
    print(f"-- attention B={B} Hq={Hq} Hkv={Hkv} L={Ln} plan={fd.attention.plan(q, kk, cfg)}", file=sys.stderr, flush=True)
    fd.decode_attention(q, kk, kk, cfg, "async")
    torch.cuda.synchronize()
    del kk
