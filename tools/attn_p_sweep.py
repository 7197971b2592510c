"""Dev tool: in-graph attention time vs explicit chunk count p on the small
decode shapes (one wave of CTAs), early PDL trigger on/off via
FDPP_ATTN_EARLY_TRIGGER in the environment."""
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
for name, B, Hq, Hkv, L in (("configs0 MHA B1 L1K", 1, 32, 32, 1024), ("70B t8 rank", 32, 8, 1, 1024),
                            ("70B t4 rank", 32, 16, 2, 1024), ("GLM MQA B8 L4K", 8, 32, 2, 4096),
                            ("GLM MQA B8 L32K", 8, 32, 2, 32768)):
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((B, Hq, 128), generator=g, device="cuda").half()
    out = torch.empty_like(q)
    kvbytes = 2 * B * Hkv * L * 128 * 2
    nrot = max(2, min(8, int(1.0e9 // kvbytes)))
    kvs = [(torch.randn((B, Hkv, L, 128), generator=g, device="cuda").half(),
            torch.randn((B, Hkv, L, 128), generator=g, device="cuda").half()) for _ in range(nrot)]
    byt = kvbytes + 2 * B * Hq * 128 * 2
    row = {}
    for p in ("auto", 2, 4, 8, 16):
        cfg = (fd.AttentionConfig.auto(1 / math.sqrt(128), cal) if p == "auto"
               else fd.AttentionConfig(p=p, scale=1 / math.sqrt(128), calib=cal))
        if p != "auto" and L // p < 128:
            continue
        fns = [lambda k=k, v=v: fd.decode_attention(q, k, v, cfg, "async", out=out, kv_prefetch=True)
               for k, v in kvs]
        t = bench._rotating_graph_time(torch, fns, reps=10)
        row[str(p) if p != "auto" else f"auto(p={fd.attention.plan(q, kvs[0][0], cfg)[0]})"] = (
            round(t * 1e6, 2), round(byt / t / 1e9 / peak, 3))
    print(json.dumps({"shape": name, "early_trigger": os.environ.get("FDPP_ATTN_EARLY_TRIGGER", "1"), **row}),
          flush=True)
    del kvs
