"""Dev tool for ncu (round 2): one launch of each shipped kernel kind the
round-2 evidence needs, on the decode shapes:
  attention MHA async (7B step shape B=32, L=1K, auto plan: cluster join, one launch)
  attention GQA/MQA tensor-core async (ChatGLM2 B=8, L=32K)
  ImplA gemv_kernel M=1 [12288,4096]; gemv_fused_kernel M=1 (QKV fused: RMSNorm + RoPE)
  ImplB cluster M=32 [4096,4096] (the O projection)
  ImplC M=128 / M=256 [12288,4096] (128- / 256-token tiles)
Each kernel is launched 3x on rotating operands; profile with
  ncu --set full -k regex:<name> -c 1 python tools/prof_r2.py
"""
import importlib
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_01282_b200 as fd  # noqa: E402
from paper_2311_01282_b200 import gemm  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
what = sys.argv[1] if len(sys.argv) > 1 else "all"
g = torch.Generator(device="cuda").manual_seed(0)
cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)

if what in ("all", "attn"):
    for B, Hq, Hkv, L in ((32, 32, 32, 1024), (8, 32, 2, 32768)):
        q = torch.randn((B, Hq, 128), generator=g, device="cuda").half()
        kv = [(torch.randn((B, Hkv, L, 128), generator=g, device="cuda").half(),
               torch.randn((B, Hkv, L, 128), generator=g, device="cuda").half()) for _ in range(2)]
        cfg = fd.AttentionConfig.auto(1 / math.sqrt(128), cal)
        for k, v in kv:
            fd.decode_attention(q, k, v, cfg, "async", kv_prefetch=True)
        del kv
if what in ("all", "gemm"):
    for n, k, cases in ((12288, 4096, ((1, D.KernelChoice.IMPL_A), (128, D.KernelChoice.IMPL_C),
                                       (256, D.KernelChoice.IMPL_C))),
                        (4096, 4096, ((32, D.KernelChoice.IMPL_B),))):
        ws = [fd.PackedWeight((torch.randn((n, k), generator=g, device="cuda") / k ** 0.5).half(), k, n)
              for _ in range(3)]
        for m, ch in cases:
            a = torch.randn((m, k), generator=g, device="cuda").half()
            for w in ws:
                D.run_device(ch, a, w)
        del ws
if what == "gemm_gu":
    # ImplB M=32 on the fused gate|up shape [22016, 4096]: one CTA per tile (staggered k order)
    n, k = 22016, 4096
    ws = [fd.PackedWeight((torch.randn((n, k), generator=g, device="cuda") / k ** 0.5).half(), k, n)
          for _ in range(3)]
    a = torch.randn((32, k), generator=g, device="cuda").half()
    for w in ws:
        D.run_device(D.KernelChoice.IMPL_B, a, w)
if what in ("all", "gemv_fused"):
    # the fused-GEMV QKV (folded RMSNorm + RoPE + KV append), Llama-2-7B shapes, M = 1
    H, Hq, Hkv = 4096, 32, 32
    x = torch.randn((1, H), generator=g, device="cuda").half()
    ssq = (x.float() ** 2).sum(1).view(1, 1).contiguous()
    pq = gemm.permute_qkv_for_gemv(gemm.PackedWeight(
        (torch.randn(((Hq + 2 * Hkv) * 128, H), generator=g, device="cuda") / 64).half(), H, (Hq + 2 * Hkv) * 128))
    kc = torch.zeros((1, Hkv, 64, 128), dtype=torch.half, device="cuda")
    vc = torch.zeros_like(kc)
    qo = torch.zeros((1, Hq, 128), dtype=torch.half, device="cuda")
    pos = torch.tensor([3], dtype=torch.int32, device="cuda")
    for _ in range(3):
        gemm.run_fused(x, pq, x_op=3, ssq_in=ssq, ssq_tiles=1, eps=1e-5, impl="A",
                       rope={"q_out": qo, "k_cache": kc, "v_cache": vc, "pos": pos})
torch.cuda.synchronize()
print("done")
