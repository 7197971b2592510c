"""ImplB time vs ring depth (default ~100 KB, 2 CTAs/SM, vs stages=8: ~200 KB,
1 CTA/SM) on the Llama-7B decode shapes; L2-cold CUDA-event timing."""
import torch

from paper_2311_01282_b200 import gemm as G
from paper_2311_01282_b200.timing import measure

torch.manual_seed(0)
for N, K in ((22016, 4096), (12288, 4096), (4096, 4096), (4096, 11008), (32000, 4096)):
    b = (torch.randn(K, N, device="cuda") / K ** 0.5).half()
    pw = G.pack_weight(b)
    for M in (1, 32, 64):
        a = torch.randn(M, K, device="cuda").half()
        row = []
        ref = None
        for st in (0, 8):
            out = G.run(G.IMPL_B, a, pw, stages=st)
            if ref is None:
                ref = out.clone()
            assert torch.equal(out, ref), "ring depth changed the result"
            t = measure(lambda: G.run(G.IMPL_B, a, pw, stages=st), reps=30, warmup=3)
            row.append(float(sorted(t)[len(t) // 2]) * 1e6)
        print(f"[{N},{K}] M={M:2d} stages=auto {row[0]:6.2f} us  stages=deep {row[1]:6.2f} us", flush=True)
