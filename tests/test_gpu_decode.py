"""The decode step (caller of the hot path): the fused GEMM
prologues/epilogues against the standalone glue kernels, the fused step
against the unfused step, and graph replay against eager execution."""

import importlib
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def mods():
    import paper_2311_01282_b200 as fd
    from paper_2311_01282_b200 import _lib, gemm, llama
    D = importlib.import_module("paper_2311_01282_b200.dispatch")
    return fd, _lib, gemm, llama, D


def _rel(a, b):
    a = a.float().cpu().numpy().reshape(a.shape[0], -1)
    b = b.float().cpu().numpy().reshape(b.shape[0], -1)
    return float((np.abs(a - b).max(axis=1) / np.maximum(np.abs(b).max(axis=1), 1e-8)).max())


def test_fused_rmsnorm_prologue_and_ssq_epilogue(torch, mods):
    fd, _lib, gemm, _, D = mods
    B, H, N = 8, 4096, 12288
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((B, H), generator=g, device="cuda").half()
    w_ln = (1 + 0.1 * torch.randn(H, generator=g, device="cuda")).half()
    pw = gemm.PackedWeight((torch.randn((N, H), generator=g, device="cuda") / 64).half(), H, N)
    # producer side: a residual GEMM whose epilogue emits the row sums of squares
    po = gemm.PackedWeight((torch.randn((H, H), generator=g, device="cuda") / 64).half(), H, H)
    a0 = torch.randn((B, H), generator=g, device="cuda").half()
    ssq = torch.zeros((H // 128, B), dtype=torch.float32, device="cuda")
    xr = x.clone()
    gemm.run_fused(a0, po, out=xr, residual=xr, ssq_out=ssq)
    ref_x = D.run_device(D.KernelChoice.IMPL_B, a0, po, residual=x)
    assert torch.equal(xr, ref_x)                       # same reduction path, bitwise
    assert torch.allclose(ssq.sum(0), xr.float().pow(2).sum(1), rtol=1e-5, atol=1e-3)
    # consumer side: RMSNorm fused into the activation tile
    out = gemm.run_fused(xr, pw, x_op=1, ssq_in=ssq, ssq_tiles=H // 128, norm_w=w_ln, eps=1e-5)
    h = torch.empty_like(xr)
    lib = _lib.load()
    _lib.check(lib.fdpp_rmsnorm(xr.data_ptr(), w_ln.data_ptr(), h.data_ptr(), B, H, 1e-5, 0,
                                _lib.stream_handle()))
    ref = D.run_device(D.KernelChoice.IMPL_B, h, pw)
    assert _rel(out, ref) <= 2e-3


def test_folded_rmsnorm_epilogue(torch, mods):
    fd, _lib, gemm, llama, D = mods
    B, H, N = 8, 4096, 22016
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((B, H), generator=g, device="cuda").half()
    w_ln = (1 + 0.1 * torch.randn(H, generator=g, device="cuda")).half()
    pw = gemm.PackedWeight((torch.randn((N, H), generator=g, device="cuda") / 64).half(), H, N)
    ssq = x.float().pow(2).sum(1)[None, :].contiguous()            # one "tile"
    out = gemm.run_fused(x, llama.fold_norm(pw, w_ln), x_op=3, ssq_in=ssq, ssq_tiles=1, eps=1e-5)
    h = torch.empty_like(x)
    lib = _lib.load()
    _lib.check(lib.fdpp_rmsnorm(x.data_ptr(), w_ln.data_ptr(), h.data_ptr(), B, H, 1e-5, 0,
                                _lib.stream_handle()))
    ref = D.run_device(D.KernelChoice.IMPL_B, h, pw)
    assert _rel(out, ref) <= 3e-3


def test_fused_silu_prologue(torch, mods):
    fd, _lib, gemm, _, D = mods
    B, F, H = 16, 11008, 4096
    g = torch.Generator(device="cuda").manual_seed(1)
    gu = torch.randn((B, 2 * F), generator=g, device="cuda").half()
    pw = gemm.PackedWeight((torch.randn((H, F), generator=g, device="cuda") / 100).half(), F, H)
    res = torch.randn((B, H), generator=g, device="cuda").half()
    out = res.clone()
    gemm.run_fused(gu, pw, out=out, residual=out, x_op=2)
    act = torch.empty((B, F), dtype=torch.half, device="cuda")
    lib = _lib.load()
    _lib.check(lib.fdpp_silu_mul(gu.data_ptr(), act.data_ptr(), B, F, 0, _lib.stream_handle()))
    ref = D.run_device(D.KernelChoice.IMPL_B, act, pw, residual=res)
    assert torch.equal(out, ref)        # identical activation bits, identical GEMM path


@pytest.mark.parametrize("B", [48, 64])
def test_fused_rmsnorm_silu_pair(torch, mods, B):
    """gate|up at 33-64 tokens (folded RMSNorm + SiLU.up) on the CTA-pair kernel
    (the flat tile's M-dependent cost, profiles/r2/flat_gemm_pair_probe.txt):
    against an fp32 restatement, output rounded like the unfused buffer."""
    fd, _lib, gemm, _, D = mods
    H, F = 4096, 11008
    g = torch.Generator(device="cuda").manual_seed(B + 1)
    x = torch.randn((B, H), generator=g, device="cuda").half()
    w = (torch.randn((2 * F, H), generator=g, device="cuda") / math.sqrt(H)).half()
    pw = gemm.interleave_gate_up(fd.PackedWeight(w, H, 2 * F))
    ssq = (x.float() ** 2).sum(1).view(1, B).contiguous()
    act = torch.empty((B, F), device="cuda", dtype=torch.half)
    gemm.run_fused(x, pw, x_op=3, ssq_in=ssq, ssq_tiles=1, eps=1e-5, silu_out=act)
    torch.cuda.synchronize()
    inv = torch.rsqrt(ssq[0] / H + 1e-5)
    y = ((x.float() @ w.float().t()) * inv[:, None]).half().float()
    gate, up = y[:, :F], y[:, F:]
    ref = (gate / (1 + torch.exp(-gate)) * up).half()
    assert _rel(act, ref) <= 2e-3
    act2 = torch.empty_like(act)
    gemm.run_fused(x, pw, x_op=3, ssq_in=ssq, ssq_tiles=1, eps=1e-5, silu_out=act2)
    assert torch.equal(act, act2)   # bitwise rerun


def test_fused_rope_append_epilogue(torch, mods):
    fd, _lib, gemm, _, D = mods
    B, H, Hq, Hkv, Dh, Lmax = 4, 4096, 32, 32, 128, 40
    g = torch.Generator(device="cuda").manual_seed(2)
    h = torch.randn((B, H), generator=g, device="cuda").half()
    N = (Hq + 2 * Hkv) * Dh
    pw = gemm.PackedWeight((torch.randn((N, H), generator=g, device="cuda") / 64).half(), H, N)
    pos = torch.tensor([3, 17, 0, 39], dtype=torch.int32, device="cuda")
    kc = torch.zeros((B, Hkv, Lmax, Dh), dtype=torch.half, device="cuda")
    vc = torch.zeros_like(kc)
    q = torch.zeros((B, Hq, Dh), dtype=torch.half, device="cuda")
    gemm.run_fused(h, pw, rope={"q_out": q, "k_cache": kc, "v_cache": vc, "pos": pos, "theta": 10000.0})
    qkv = D.run_device(D.KernelChoice.IMPL_B, h, pw, ctas=-2)     # same cluster split
    kc2, vc2, q2 = torch.zeros_like(kc), torch.zeros_like(vc), torch.zeros_like(q)
    lib = _lib.load()
    _lib.check(lib.fdpp_rope_append(qkv.data_ptr(), q2.data_ptr(), kc2.data_ptr(), vc2.data_ptr(),
                                    pos.data_ptr(), B, Hq, Hkv, Dh, kc2.stride(0), kc2.stride(1),
                                    10000.0, 0, _lib.stream_handle()))
    assert torch.equal(q, q2) and torch.equal(kc, kc2) and torch.equal(vc, vc2)


def _decoder(torch, mods, fused, layers=2, B=4, L=64):
    fd, _lib, gemm, llama, D = mods
    table = D.DispatchTable(fingerprint="test")
    for n, k in llama.LLAMA2_7B.gemm_shapes().values():
        table.add(D.DispatchEntry(n=n, k=k, m1=1, m2=128))
    dec = llama.LlamaDecoder(llama.LLAMA2_7B, B, L + 8, table=table, seed=5, n_layers=layers,
                             fused=fused)
    dec.prefill_random(L, seed=6)
    return dec


def test_fused_step_matches_unfused_step(torch, mods):
    a = _decoder(torch, mods, fused=True)
    b = _decoder(torch, mods, fused=False)
    a.enqueue_step()
    b.enqueue_step()
    torch.cuda.synchronize()
    assert _rel(a.logits, b.logits) <= 2e-2
    for li in range(a.n_layers):
        assert _rel(a.k_cache[li][:, :, 64], b.k_cache[li][:, :, 64]) <= 2e-2
    # graph replay == eager for the next step
    a.capture()
    s0 = a.pos.clone()
    a.step()
    torch.cuda.synchronize()
    assert torch.equal(a.pos, s0 + 1)


def _tiny_weights(torch, cfg, seed=0):
    g = torch.Generator().manual_seed(seed)

    def w(n, k):
        return torch.randn((n, k), generator=g) / math.sqrt(k)

    D = cfg.head_dim
    layers = [{"qkv": w((cfg.n_heads + 2 * cfg.n_kv_heads) * D, cfg.hidden),
               "o": w(cfg.hidden, cfg.n_heads * D), "gate_up": w(2 * cfg.ffn, cfg.hidden),
               "down": w(cfg.hidden, cfg.ffn),
               "ln1": 1 + 0.1 * torch.randn(cfg.hidden, generator=g),
               "ln2": 1 + 0.1 * torch.randn(cfg.hidden, generator=g)} for _ in range(cfg.n_layers)]
    return {"layers": layers, "embed": torch.randn((cfg.vocab, cfg.hidden), generator=g),
            "lm_head": w(cfg.vocab, cfg.hidden), "ln_f": 1 + 0.1 * torch.randn(cfg.hidden, generator=g)}


@pytest.mark.parametrize("n_kv,B,m1,dt", [(4, 4, 1, "float16"), (1, 4, 1, "float16"), (4, 2, 3, "float16"),
                                          (1, 4, 1, "bfloat16")])  # ImplB; G = 8; fused GEMV; bf16
def test_decode_step_matches_fp32_reference(torch, mods, n_kv, B, m1, dt):
    """The whole fused decode step (folded RMSNorm, RoPE + KV append epilogue,
    async attention, residual epilogues, SiLU*up) against tp.reference_layer
    in fp32 on the same weights, KV state and tokens."""
    from paper_2311_01282_b200 import tp
    fd, _lib, gemm, llama, D = mods
    cfg = llama.LlamaConfig("tiny", hidden=1024, n_heads=8, n_kv_heads=n_kv, head_dim=128, ffn=1536,
                            n_layers=2, vocab=512)
    W = _tiny_weights(torch, cfg)
    table = D.DispatchTable(fingerprint="test")
    for n, k in cfg.gemm_shapes().values():
        table.add(D.DispatchEntry(n=n, k=k, m1=m1, m2=128))
    L = 200
    dtype = getattr(torch, dt)
    dec = llama.LlamaDecoder(cfg, B, L + 8, table=table, weights=W, gemv_step=m1 > B, dtype=dtype)
    assert dec.fused and dec.step_impl == ("A" if m1 > B else "B")
    dec.prefill_random(L, seed=3)
    x = W["embed"][dec.ids.long().cpu()].to(dtype).float()
    kc = [k.float().cpu() for k in dec.k_cache]
    vc = [v.float().cpu() for v in dec.v_cache]
    pos = dec.pos.long().cpu()
    for li in range(cfg.n_layers):
        Lw = {k: v.to(dtype).float() for k, v in W["layers"][li].items()}
        x = tp.reference_layer(x, Lw, kc[li], vc[li], pos, pos + 1, cfg, cfg.n_heads, cfg.n_kv_heads)
    dec.enqueue_step()
    torch.cuda.synchronize()
    assert int(dec.recomputed.item()) == 0
    assert _rel(dec.x, x) <= (2e-2 if dt == "float16" else 6e-2)  # bf16: 8-bit mantissa activations
    for li in range(cfg.n_layers):  # appended K rows (RoPE'd in the QKV epilogue)
        got = dec.k_cache[li][torch.arange(B), :, pos.cuda()].float().cpu()
        exp = kc[li][torch.arange(B), :, pos]
        assert _rel(got, exp) <= (2e-2 if dt == "float16" else 6e-2)


def test_row_ssq(torch, mods):
    fd, _lib, *_ = mods
    x = torch.randn((5, 4096), device="cuda").half()
    out = torch.empty(5, device="cuda")
    _lib.check(_lib.load().fdpp_row_ssq(x.data_ptr(), out.data_ptr(), 5, 4096, 0, _lib.stream_handle()))
    torch.cuda.synchronize()
    ref = (x.float() ** 2).sum(1)
    assert torch.allclose(out, ref, rtol=1e-5)


def test_fused_silu_epilogue(torch, mods):
    """gate|up GEMM with the SiLU*up epilogue (tile-interleaved weight rows) ==
    the plain fused GEMM into [gate | up] followed by the silu_mul kernel."""
    fd, _lib, gemm, _, D = mods
    for B, H, F in ((32, 4096, 11008), (5, 1024, 1536), (64, 4096, 11008)):  # B = 64: the CTA-pair kernel
        g = torch.Generator(device="cuda").manual_seed(B)
        x = torch.randn((B, H), generator=g, device="cuda").half()
        w = (torch.randn((2 * F, H), generator=g, device="cuda") / math.sqrt(H)).half()
        pw = fd.PackedWeight(w, H, 2 * F)
        gu = gemm.run_fused(x, pw)
        act_ref = torch.empty((B, F), device="cuda", dtype=torch.half)
        _lib.check(_lib.load().fdpp_silu_mul(gu.data_ptr(), act_ref.data_ptr(), B, F, 0, _lib.stream_handle()))
        act = torch.empty_like(act_ref)
        gemm.run_fused(x, gemm.interleave_gate_up(pw), silu_out=act)
        torch.cuda.synchronize()
        assert _rel(act, act_ref) <= 2e-3


def test_decoder_calibrate(torch, mods):
    """LlamaDecoder.calibrate(): fits phi / band to the model's own attention
    logits, restores the decode state, and the recalibrated step flags nothing."""
    fd, _lib, gemm, llama, D = mods
    dec = _decoder(torch, mods, fused=True, layers=2, B=4, L=64)
    pos0, ids0 = dec.pos.clone(), dec.ids.clone()
    cal = dec.calibrate(samples_per_layer=8192)
    assert torch.equal(dec.pos, pos0) and torch.equal(dec.ids, ids0)
    assert cal.a < 0 < cal.b and dec.attn_cfg.calib == cal
    dec.enqueue_step()
    torch.cuda.synchronize()
    assert int(dec.recomputed.item()) == 0


@pytest.mark.parametrize("M", [1, 2])
def test_fused_gemv_matches_fused_flat_gemm(torch, mods, M):
    """fdpp_gemv_fused (ImplA form of the decode-step fusions) against the
    ImplB fused GEMM: residual + sums of squares, folded RMSNorm, RoPE + KV
    append (permuted QKV rows), SiLU*up (permuted gate|up rows)."""
    fd, _lib, gemm, _, D = mods
    g = torch.Generator(device="cuda").manual_seed(M)
    H = 1024
    x = torch.randn((M, H), generator=g, device="cuda").half()
    res = torch.randn((M, H), generator=g, device="cuda").half()
    ssq_in = (x.float() ** 2).sum(1, keepdim=True).t().contiguous()      # one tile per row
    # residual GEMM with sums of squares
    w = fd.PackedWeight((torch.randn((H, H), generator=g, device="cuda") / 32).half(), H, H)
    o_b, o_a = torch.empty_like(res), torch.empty_like(res)
    s_b = torch.zeros((H // 128, M), device="cuda")
    s_a = torch.zeros((H // 8, M), device="cuda")
    gemm.run_fused(x, w, out=o_b, residual=res, ssq_out=s_b)
    gemm.run_fused(x, w, out=o_a, residual=res, ssq_out=s_a, impl="A")
    torch.cuda.synchronize()
    assert _rel(o_a, o_b) <= 2e-3
    assert torch.allclose(s_a.sum(0), s_b.sum(0), rtol=1e-3)
    # folded RMSNorm
    f_b = gemm.run_fused(x, w, x_op=3, ssq_in=ssq_in, ssq_tiles=1)
    f_a = gemm.run_fused(x, w, x_op=3, ssq_in=ssq_in, ssq_tiles=1, impl="A")
    torch.cuda.synchronize()
    assert _rel(f_a, f_b) <= 2e-3
    # RoPE + KV append
    Hq, Hkv, Lmax = 4, 2, 16
    wq = fd.PackedWeight((torch.randn(((Hq + 2 * Hkv) * 128, H), generator=g, device="cuda") / 32).half(),
                         H, (Hq + 2 * Hkv) * 128)
    pos = torch.tensor([3, 9][:M], dtype=torch.int32, device="cuda")
    outs = []
    for impl, ww in (("B", wq), ("A", gemm.permute_qkv_for_gemv(wq))):
        q = torch.zeros((M, Hq, 128), device="cuda").half()
        kc = torch.zeros((M, Hkv, Lmax, 128), device="cuda").half()
        vc = torch.zeros_like(kc)
        gemm.run_fused(x, ww, rope={"q_out": q, "k_cache": kc, "v_cache": vc, "pos": pos}, impl=impl)
        outs.append((q, kc, vc))
    torch.cuda.synchronize()
    for a, b in zip(outs[0], outs[1]):
        assert _rel(b.reshape(M, -1), a.reshape(M, -1)) <= 2e-3
    # SiLU*up
    F = 768
    wg = fd.PackedWeight((torch.randn((2 * F, H), generator=g, device="cuda") / 32).half(), H, 2 * F)
    act_b = torch.empty((M, F), device="cuda").half()
    act_a = torch.empty_like(act_b)
    gemm.run_fused(x, gemm.interleave_gate_up(wg), silu_out=act_b)
    gemm.run_fused(x, gemm.permute_gate_up_for_gemv(wg), silu_out=act_a, impl="A")
    torch.cuda.synchronize()
    assert _rel(act_a, act_b) <= 2e-3


def test_rope_epilogue_long_positions(torch, mods):
    """RoPE + KV append at 32K-scale positions (ChatGLM2 config: L = 32K) against
    an f64-angle rotation of the plain projection (full-range sin/cos)."""
    from paper_2311_01282_b200 import tp
    fd, _lib, gemm, _, D = mods
    g = torch.Generator(device="cuda").manual_seed(9)
    M, H, Hq, Hkv = 2, 1024, 2, 1
    N = (Hq + 2 * Hkv) * 128
    x = torch.randn((M, H), generator=g, device="cuda").half()
    w = fd.PackedWeight((torch.randn((N, H), generator=g, device="cuda") / 32).half(), H, N)
    pos = torch.tensor([32767, 20001], dtype=torch.int32, device="cuda")
    plain = gemm.run_fused(x, w).float().cpu()
    for impl, ww in (("B", w), ("A", gemm.permute_qkv_for_gemv(w))):
        q = torch.zeros((M, Hq, 128), device="cuda").half()
        kc = torch.zeros((M, Hkv, 32768, 128), device="cuda").half()
        vc = torch.zeros_like(kc)
        gemm.run_fused(x, ww, rope={"q_out": q, "k_cache": kc, "v_cache": vc, "pos": pos}, impl=impl)
        torch.cuda.synchronize()
        ref_q = tp._rope(plain[:, :Hq * 128].view(M, Hq, 128), pos.cpu(), 10000.0)
        ref_k = tp._rope(plain[:, Hq * 128:(Hq + Hkv) * 128].view(M, Hkv, 128), pos.cpu(), 10000.0)
        assert _rel(q.float().cpu(), ref_q) <= 2e-3, impl
        got_k = kc[torch.arange(M), :, pos.long()].float().cpu()
        assert _rel(got_k, ref_k) <= 2e-3, impl
