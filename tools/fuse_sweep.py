"""Dev tool: in-graph per-launch time of plain vs fused ImplB variants."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200 import gemm  # noqa: E402
from tools.mode_sweep import graph_time  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
B = 32
for n, k in ((12288, 4096), (22016, 4096), (4096, 11008), (32000, 4096)):
    L = max(4, min(24, int(2.4e9 // (n * k * 2))))
    ws = [gemm.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n) for _ in range(L)]
    x = torch.randn((B, k), device="cuda").half()
    gu = torch.randn((B, 2 * k), device="cuda").half()
    out = torch.empty((B, n), device="cuda", dtype=torch.half)
    ssq = torch.ones((32, B), device="cuda")
    lnw = torch.ones(k, device="cuda").half()
    ssq_o = torch.zeros((n // 128, B), device="cuda")
    res = {}
    res["plain"] = graph_time(lambda: [D.run_device(D.KernelChoice.IMPL_B, x, w, out=out) for w in ws]) / L
    res["fused_noop"] = graph_time(lambda: [gemm.run_fused(x, w, out=out) for w in ws]) / L
    res["ssq_out"] = graph_time(lambda: [gemm.run_fused(x, w, out=out, ssq_out=ssq_o) for w in ws]) / L
    res["rmsnorm"] = graph_time(lambda: [gemm.run_fused(x, w, out=out, x_op=1, ssq_in=ssq, ssq_tiles=32,
                                                        norm_w=lnw) for w in ws]) / L
    res["silu"] = graph_time(lambda: [gemm.run_fused(gu, w, out=out, x_op=2) for w in ws]) / L
    print(f"[{n},{k}] " + "  ".join(f"{kk}={v:6.2f}us" for kk, v in res.items()), flush=True)
    del ws

# standalone glue kernels, back to back in one graph (per-launch time)
from paper_2311_01282_b200 import _lib  # noqa: E402
lib = _lib.load()
x = torch.randn((B, 4096), device="cuda").half()
h = torch.empty_like(x)
lnw = torch.ones(4096, device="cuda").half()
gu = torch.randn((B, 2 * 11008), device="cuda").half()
act = torch.empty((B, 11008), device="cuda").half()
qkv = torch.randn((B, 12288), device="cuda").half()
q = torch.empty((B, 32, 128), device="cuda").half()
kc = torch.zeros((B, 32, 64, 128), device="cuda").half()
vc = torch.zeros_like(kc)
pos = torch.full((B,), 5, dtype=torch.int32, device="cuda")
st = lambda: _lib.stream_handle()  # noqa: E731
N = 24
t_rms = graph_time(lambda: [lib.fdpp_rmsnorm(x.data_ptr(), lnw.data_ptr(), h.data_ptr(), B, 4096, 1e-5, 0, st()) for _ in range(N)]) / N
t_silu = graph_time(lambda: [lib.fdpp_silu_mul(gu.data_ptr(), act.data_ptr(), B, 11008, 0, st()) for _ in range(N)]) / N
t_rope = graph_time(lambda: [lib.fdpp_rope_append(qkv.data_ptr(), q.data_ptr(), kc.data_ptr(), vc.data_ptr(), pos.data_ptr(), B, 32, 32, 128, kc.stride(0), kc.stride(1), 10000.0, 0, st()) for _ in range(N)]) / N
print(f"glue: rmsnorm={t_rms:6.2f}us silu_mul={t_silu:6.2f}us rope_append={t_rope:6.2f}us", flush=True)
