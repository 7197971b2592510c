"""Dev tool: attention device time in-graph (rotating K/V caches > L2, like
bench.py configs[0]) over decode shapes, kv_prefetch off/on.

    python tools/attn_graph_sweep.py  -> gpurun_out/attn_graph_sweep.json
"""
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
SHAPES = [  # (name, B, Hq, Hkv, L)
    ("configs0 MHA B1 L1K", 1, 32, 32, 1024),
    ("7B MHA B32 L1K", 32, 32, 32, 1024),
    ("7B MHA B8 L1K", 8, 32, 32, 1024),
    ("70B t8 rank B32 G8 L1K", 32, 8, 1, 1024),
    ("70B t4 rank B32 G8 L1K", 32, 16, 2, 1024),
    ("70B t1 B32 G8 L1K", 32, 64, 8, 1024),
    ("GLM MQA B8 L32K", 8, 32, 2, 32768),
    ("GLM MQA B8 L4K", 8, 32, 2, 4096),
]
res = []
for name, B, Hq, Hkv, L in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(0)
    cfg = fd.AttentionConfig.auto(1 / math.sqrt(128), cal)
    q = torch.randn((B, Hq, 128), generator=g, device="cuda").half()
    out = torch.empty_like(q)
    kvbytes = 2 * B * Hkv * L * 128 * 2
    nrot = max(2, min(8, int(1.0e9 // kvbytes)))
    kvs = [(torch.randn((B, Hkv, L, 128), generator=g, device="cuda").half(),
            torch.randn((B, Hkv, L, 128), generator=g, device="cuda").half()) for _ in range(nrot)]
    byt = kvbytes + 2 * B * Hq * 128 * 2
    for pf in (False, True):
        fns = [lambda k=k, v=v: fd.decode_attention(q, k, v, cfg, "async", out=out, kv_prefetch=pf)
               for k, v in kvs]
        t = bench._rotating_graph_time(torch, fns, reps=10)
        r = {"shape": name, "B": B, "Hq": Hq, "Hkv": Hkv, "L": L, "kv_prefetch": pf,
             "plan": list(fd.attention.plan(q, kvs[0][0], cfg)),
             "launches": fd.attention.launches(q, kvs[0][0], cfg),
             "us": round(t * 1e6, 2), "gbs": round(byt / t / 1e9, 1), "frac": round(byt / t / 1e9 / peak, 3)}
        res.append(r)
        print(json.dumps(r), flush=True)
    del kvs
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "attn_graph_sweep.json"), "w"), indent=1)
