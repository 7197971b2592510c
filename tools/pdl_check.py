"""Dev tool: per-launch device time of back-to-back GEMMs in one CUDA graph,
PDL on vs off (distinct weights per launch so nothing is L2-resident)."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200 import _lib  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
lib = _lib.load()


def graph_time(fn, reps=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for n, k, m in ((4096, 4096, 32), (22016, 4096, 32), (4096, 4096, 1)):
    L = 24
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    a = torch.randn((m, k), device="cuda").half()
    out = torch.empty((m, n), device="cuda", dtype=torch.half)
    for impl in ("B", "A") if m <= 8 else ("B",):
        ch = D.KernelChoice.IMPL_B if impl == "B" else D.KernelChoice.IMPL_A
        for pdl in (1, 0):
            lib.fdpp_set_pdl(pdl)

            def fn():
                for w in ws:
                    D.run_device(ch, a, w, out=out)
            t = graph_time(fn) / L
            byt = n * k * 2
            print(f"[{n},{k}] M={m} Impl{impl} pdl={pdl}: {t:7.2f} us/launch  {byt/t/1e3:7.0f} GB/s", flush=True)
    lib.fdpp_set_pdl(1)
    del ws

# empty-ish reference: the tiny advance kernel back to back
pos = torch.zeros(32, dtype=torch.int32, device="cuda")
for pdl in (1, 0):
    lib.fdpp_set_pdl(pdl)
    t = graph_time(lambda: [lib.fdpp_advance_positions(pos.data_ptr(), None, 32, _lib.stream_handle()) for _ in range(100)]) / 100
    print(f"tiny kernel pdl={pdl}: {t:6.2f} us/launch", flush=True)
lib.fdpp_set_pdl(1)
