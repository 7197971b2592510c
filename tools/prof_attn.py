"""Dev tool for ncu: decode attention at the bench shape (B=32, H=32, L=1024+)."""
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402

B, H, L, D = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (32, 32, 1040, 128)))
Hkv = int(sys.argv[5]) if len(sys.argv) > 5 else H
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
cfg = fd.AttentionConfig.auto(1 / math.sqrt(D), cal)
caches = []
for i in range(3):
    k = torch.randn((B, Hkv, L, D), device="cuda").half()
    v = torch.randn((B, Hkv, L, D), device="cuda").half()
    caches.append((k, v))
q = torch.randn((B, H, D), device="cuda").half()
out = torch.empty_like(q)
print("plan", fd.attention.plan(q, caches[0][0], cfg))
for i in range(reps):
    k, v = caches[i % 3]
    fd.decode_attention(q, k, v, cfg, "async", out=out)
torch.cuda.synchronize()
print("done")
