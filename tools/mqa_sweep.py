"""Dev tool: device time of async decode attention for GQA/MQA shapes (ChatGLM2 config 4)."""
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200.timing import measure, median_mad  # noqa: E402

cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
D = 128
for B, Hq, Hkv, L in ((8, 32, 2, 32768), (32, 8, 1, 1024), (32, 16, 2, 1024), (32, 64, 8, 1024), (8, 8, 1, 32768)):
    k = torch.randn((B, Hkv, L, D), device="cuda").half()
    v = torch.randn((B, Hkv, L, D), device="cuda").half()
    q = torch.randn((B, Hq, D), device="cuda").half()
    out = torch.empty_like(q)
    byt = B * Hkv * L * D * 4 + 2 * B * Hq * D * 2
    for p, spc in ((0, 0), (2, 1), (4, 1), (8, 1), (16, 1), (20, 1), (24, 1), (27, 1), (32, 1)):
        cfg = fd.AttentionConfig(p=p or "auto", scale=1 / math.sqrt(D), calib=cal, splits_per_chunk=spc)
        plan = fd.attention.plan(q, k, cfg)
        med, _ = median_mad(measure(lambda: fd.decode_attention(q, k, v, cfg, "async", out=out), reps=10, warmup=2))
        print(f"B={B} Hq={Hq} Hkv={Hkv} L={L} p={p} plan={plan} {med*1e6:8.1f} us {byt/med/1e9:7.0f} GB/s", flush=True)
    del k, v
