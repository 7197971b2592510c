"""Dev probe: configs[0] attention (B=1, 32 heads, L=1K) in-graph, 8 rotating
caches, programmatic dependent launch on vs off (fdpp_set_pdl), kv_prefetch
on/off: does consecutive-attention overlap happen at all?"""
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
cfg = fd.AttentionConfig.auto(1 / math.sqrt(128), cal)
lib = _lib.load()
for pdl in (1, 0):
    lib.fdpp_set_pdl(pdl)
    for pf in (True, False):
        fns = [lambda k=k, v=v: fd.decode_attention(q, k, v, cfg, "async", out=out, kv_prefetch=pf) for k, v in kvs]
        t = bench._rotating_graph_time(torch, fns, reps=20)
        print(f"pdl={pdl} kv_prefetch={pf}: {t * 1e6:.2f} us per call", flush=True)
lib.fdpp_set_pdl(1)

# the same question for the flat GEMM (cluster split-K, [4096, 4096], M = 32) and
# for the decode step as a whole
D = __import__("importlib").import_module("paper_2311_01282_b200.dispatch")
ws = [fd.PackedWeight((torch.randn((4096, 4096), device="cuda") / 64).half(), 4096, 4096) for _ in range(8)]
a = torch.randn((32, 4096), device="cuda").half()
o = torch.empty((32, 4096), device="cuda", dtype=torch.half)
for pdl in (1, 0):
    lib.fdpp_set_pdl(pdl)
    t = bench._rotating_graph_time(torch, [lambda w=w: D.run_device(D.KernelChoice.IMPL_B, a, w, out=o) for w in ws], reps=20)
    print(f"pdl={pdl} ImplB [4096,4096] M=32: {t * 1e6:.2f} us per call", flush=True)
lib.fdpp_set_pdl(1)
