"""Dev probe: does PDL overlap consecutive attention launches when they are
not cluster launches?  configs[0] shape, cluster plan (auto) vs global-join
plan (p=8, 2 splits per chunk), PDL on/off."""
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200 import _lib  # noqa: E402

cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
g = torch.Generator(device="cuda").manual_seed(0)
B, H, L = 1, 32, 1024
q = torch.randn((B, H, 128), generator=g, device="cuda").half()
out = torch.empty_like(q)
kvs = [(torch.randn((B, H, L, 128), generator=g, device="cuda").half(),
        torch.randn((B, H, L, 128), generator=g, device="cuda").half()) for _ in range(8)]
lib = _lib.load()
for name, cfg in (("cluster auto", fd.AttentionConfig.auto(1 / math.sqrt(128), cal)),
                  ("global p=8x2", fd.AttentionConfig(p=8, scale=1 / math.sqrt(128), calib=cal, splits_per_chunk=2)),
                  ("global p=4x4", fd.AttentionConfig(p=4, scale=1 / math.sqrt(128), calib=cal, splits_per_chunk=4))):
    for pdl in (1, 0):
        lib.fdpp_set_pdl(pdl)
        fns = [lambda k=k, v=v: fd.decode_attention(q, k, v, cfg, "async", out=out, kv_prefetch=True) for k, v in kvs]
        t = bench._rotating_graph_time(torch, fns, reps=20)
        print(f"{name:14s} launches={fd.attention.launches(q, kvs[0][0], cfg)} pdl={pdl}: {t * 1e6:.2f} us per call",
              flush=True)
lib.fdpp_set_pdl(1)
