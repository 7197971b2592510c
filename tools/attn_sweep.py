"""Dev tool: device time of async decode attention over (B, L, splits)."""
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200.timing import measure, median_mad  # noqa: E402

cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
H, D = 32, 128
shapes = ((1, 1024), (1, 8192), (8, 4096), (32, 1040), (32, 4096))
if len(sys.argv) > 1:
    shapes = tuple(tuple(int(x) for x in s.split("x")) for s in sys.argv[1].split(","))
for B, L in shapes:
    caches = []
    nrot = max(1, min(4, int(400e6 // (B * H * L * D * 4))))
    for i in range(nrot):
        caches.append((torch.randn((B, H, L, D), device="cuda").half(),
                       torch.randn((B, H, L, D), device="cuda").half()))
    q = torch.randn((B, H, D), device="cuda").half()
    out = torch.empty_like(q)
    byt = B * H * L * D * 4 + 2 * B * H * D * 2
    for p, spc in ((0, 0), (1, 1), (2, 1), (3, 1), (4, 1), (6, 1), (8, 1), (1, 2), (1, 4)):
        cfg = fd.AttentionConfig(p=p or "auto", scale=1 / math.sqrt(D), calib=cal, splits_per_chunk=spc)
        it = [0]

        def f():
            k, v = caches[it[0] % nrot]
            it[0] += 1
            fd.decode_attention(q, k, v, cfg, "async", out=out)
        plan = fd.attention.plan(q, caches[0][0], cfg)
        med, _ = median_mad(measure(f, reps=10, warmup=2))
        print(f"B={B:3d} L={L:5d} p={p} spc={spc:2d} plan={plan} {med*1e6:8.1f} us {byt/med/1e9:7.0f} GB/s",
              flush=True)
    del caches
