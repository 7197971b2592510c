"""Dev tool: in-graph MHA attention time vs chunk count p (decode shapes,
32 heads x 128, fp16), to re-check the wave-aware split planner."""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2311_01282_b200 as fd  # noqa: E402

peak, _ = bench._peaks()
cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
for B, L in ((1, 1024), (2, 1024), (4, 1024), (1, 4096)) if len(sys.argv) > 1 else ((4, 1024), (8, 1024), (16, 1024), (32, 1024), (8, 4096), (16, 4096)):
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((B, 32, 128), generator=g, device="cuda").half()
    out = torch.empty_like(q)
    kvbytes = 2 * B * 32 * L * 128 * 2
    nrot = max(2, min(8, int(1.0e9 // kvbytes)))
    kvs = [(torch.randn((B, 32, L, 128), generator=g, device="cuda").half(),
            torch.randn((B, 32, L, 128), generator=g, device="cuda").half()) for _ in range(nrot)]
    byt = kvbytes + 2 * B * 32 * 128 * 2
    row = {"B": B, "L": L}
    for p in ["auto"] + list(range(1, 17)):
        cfg = (fd.AttentionConfig.auto(1 / math.sqrt(128), cal) if p == "auto"
               else fd.AttentionConfig(p=p, scale=1 / math.sqrt(128), calib=cal, splits_per_chunk=1))
        fns = [lambda k=k, v=v: fd.decode_attention(q, k, v, cfg, "async", out=out, kv_prefetch=True) for k, v in kvs]
        t = bench._rotating_graph_time(torch, fns, reps=10)
        key = f"auto(p={fd.attention.plan(q, kvs[0][0], cfg)[0]})" if p == "auto" else str(p)
        row[key] = (round(t * 1e6, 2), round(byt / t / 1e9 / peak, 3))
    print(json.dumps(row), flush=True)
    del kvs
