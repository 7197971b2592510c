"""Dev tool: one attention case (argv: B Hq Hkv L p inject_mode), prints flags
and error vs the oracle; run under `timeout` with FDPP_ATTN_ABORT=0/1."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_01282_b200 as fd  # noqa: E402
from oracle import flatdecode_oracle as O  # noqa: E402

B, Hq, Hkv, L, p = (int(x) for x in sys.argv[1:6])
mode = sys.argv[6]
spc = int(sys.argv[7]) if len(sys.argv) > 7 else 0
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn((B, Hq, 128), generator=g, device="cuda").half()
k = torch.randn((B, Hkv, L, 128), generator=g, device="cuda").half()
v = torch.randn((B, Hkv, L, 128), generator=g, device="cuda").half()
if mode == "q":
    q[0, Hq // 3] = (q[0, Hq // 3].float() * 12).half()
elif mode == "k":
    k[0, 0, L // 2].mul_(40.0)
cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
cfg = fd.AttentionConfig(p=p, scale=1 / math.sqrt(128), calib=cal, splits_per_chunk=spc) if p > 0 else fd.AttentionConfig.auto(1 / math.sqrt(128), cal)
print("plan", fd.attention.plan(q, k, cfg), "launches", fd.attention.launches(q, k, cfg), flush=True)
o, st = fd.decode_attention(q, k, v, cfg, "async")
torch.cuda.synchronize()
print("kernel done, rows", st.rows_recomputed, flush=True)
pp = fd.attention.plan(q, k, cfg)[0]
G = Hq // Hkv
bad = 0
for b in range(B):
    for h in range(Hkv):
        ref, _, redo = O.batch_decode_attention(q[b, h * G:(h + 1) * G].float().cpu().numpy(), k[b, h].float().cpu().numpy(),
                                                v[b, h].float().cpu().numpy(), pp, cfg.scale, O.Calib(cal.phi, cal.a, cal.b), "async")
        got = st.row_mask[b, h * G:(h + 1) * G].cpu().numpy()
        err = O.rel_error_rowwise(o[b, h * G:(h + 1) * G].float().cpu().numpy(), ref)
        if not np.array_equal(got, redo) or err > 2e-3:
            bad += 1
            print("MISMATCH", b, h, got.astype(int), redo.astype(int), err)
print("OK" if bad == 0 else f"{bad} bad groups", flush=True)
