"""Dev tool: per-CTA timeline of one async attention launch (trace build:
nvcc -DFDPP_ATRACE, tools/atrace_build.sh).  Prints, relative to the first
CTA entry, percentiles of: entry, after pdl_wait, setup done, consumers'
main loop done, partial published, ticket resolved, join done, producer done."""
import ctypes
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_01282_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath("tools/atrace/libfdpp.so")
import paper_2311_01282_b200 as fd  # noqa: E402

lib = _lib.load()
lib.fdpp_atrace_read.argtypes = [ctypes.c_void_p]
B, Hq, Hkv, L = (int(x) for x in sys.argv[1:5])
D = 128
cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
cfg = fd.AttentionConfig.auto(1 / math.sqrt(D), cal)
q = torch.randn((B, Hq, D), device="cuda").half()
k = torch.randn((B, Hkv, L, D), device="cuda").half()
v = torch.randn((B, Hkv, L, D), device="cuda").half()
out = torch.empty_like(q)
for _ in range(3):
    fd.decode_attention(q, k, v, cfg, "async", out=out)
torch.cuda.synchronize()
lib.fdpp_atrace_reset()
# back-to-back calls so the clocks are at their loaded level: the buffer keeps the
# last call's stamps (plain stores overwrite; the max-slots only grow)
for _ in range(int(os.environ.get("ATRACE_CALLS", "300"))):
    fd.decode_attention(q, k, v, cfg, "async", out=out)
torch.cuda.synchronize()
buf = np.zeros((8192, 8), dtype=np.uint64)
lib.fdpp_atrace_read(buf.ctypes.data)
t = buf.astype(np.int64)
ok = t[:, 0] > 0
t = t[ok]
base = t[:, 0].min()
names = ["entry", "pdl_done", "setup", "published", "ticket/cluster_synced", "joined", "consumers_done", "producer_done"]
print(f"B={B} Hq={Hq} Hkv={Hkv} L={L} plan={fd.attention.plan(q, k, cfg)} CTAs={len(t)}  (us from first entry)")
for j, nm in enumerate(names):
    col = t[:, j]
    col = col[col > 0]
    if len(col) == 0:
        continue
    r = (col - base) / 1000.0
    print(f"  {nm:15s} n={len(col):5d}  min={r.min():7.2f}  p50={np.median(r):7.2f}  p90={np.percentile(r, 90):7.2f}  max={r.max():7.2f}")
