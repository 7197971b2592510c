"""Dev tool: in-graph per-launch time of ImplB modes per decode shape."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200 import _lib  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")


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


Ms = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 32]
for n, k in ((12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (32000, 4096)):
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    for m in Ms:
        a = torch.randn((m, k), device="cuda").half()
        out = torch.empty((m, n), device="cuda", dtype=torch.half)
        res = []
        modes = [("auto", D.KernelChoice.IMPL_B, 0), ("sk148", D.KernelChoice.IMPL_B, 148),
                 ("sk296", D.KernelChoice.IMPL_B, 296), ("cl2", D.KernelChoice.IMPL_B, -2),
                 ("cl4", D.KernelChoice.IMPL_B, -4), ("cl8", D.KernelChoice.IMPL_B, -8)]
        if m <= 8:
            modes.append(("gemv", D.KernelChoice.IMPL_A, 0))
        for name, ch, ctas in modes:
            t = graph_time(lambda: [D.run_device(ch, a, w, out=out, ctas=ctas) for w in ws]) / L
            res.append(f"{name}={t:6.2f}us/{n*k*2/t/1e3:5.0f}")
        print(f"[{n},{k}] M={m:2d} " + "  ".join(res), flush=True)
    del ws
