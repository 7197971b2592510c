"""Dev tool: cross-launch timeline of back-to-back tcgen05 GEMMs (trace build)."""
import ctypes
import importlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_01282_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath("tools/trace/libfdpp.so")
import paper_2311_01282_b200 as fd  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
lib = _lib.load()
lib.fdpp_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
n, k, m = (int(x) for x in sys.argv[1:4])
pdl = int(sys.argv[4]) if len(sys.argv) > 4 else 1
lib.fdpp_set_pdl(pdl)
NL = 8
ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(NL)]
a = torch.randn((m, k), device="cuda").half()
out = torch.empty((m, n), device="cuda", dtype=torch.half)


def fn():
    for w in ws:
        D.run_device(D.KernelChoice.IMPL_B, a, w, out=out)


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    fn()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    fn()
torch.cuda.synchronize()
lib.fdpp_trace_reset()
g.replay()
torch.cuda.synchronize()
buf = np.zeros((8, 512, 8), dtype=np.uint64)
lib.fdpp_trace_read(buf.ctypes.data, 0)
t = buf.astype(np.int64)
G = 148
base = t[0, :G, 7][t[0, :G, 7] > 0].min()
names = ["entry", "start", "W issued", "pdl done", "1st full", "last full", "last tmem_full", "end"]
order = [7, 0, 1, 2, 3, 4, 5, 6]
print(f"pdl={pdl}  [{n},{k}] M={m}: times in us relative to launch-0 first entry")
for L in range(NL):
    row = t[L, :G]
    ok = row[:, 7] > 0
    if not ok.any():
        continue
    r = (row[ok] - base) / 1000.0
    cells = [f"{nm}={r[:, j].min():6.2f}/{np.median(r[:, j]):6.2f}/{r[:, j].max():6.2f}" for nm, j in zip(names, order)]
    print(f"L{L}: " + "  ".join(cells[:2] + cells[3:4] + cells[5:]))
