"""Device GEMM plumbing shared by flatgemm.py and dispatch.py.

C[M,N] = A[M,K] · B[K,N] with B prepacked once into W[N, ldw] (K-major, the
layout both the GEMV and the tcgen05 TMA tiles stream).  fp16/bf16 operands
run on the tensor-core / GEMV hot path (fp32 accumulation, the north_star's
2e-3 bar); float32 operands -- the reference API's numpy f32 arrays or f32
CUDA tensors -- run the f32 CUDA-core forms of the same three impls
(csrc/gemm_f32.cu), keeping the reference's own <= 1e-4 contract.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib, workspace
from .matrix import ShapeError

IMPL_A, IMPL_B, IMPL_C = _lib.IMPL_A, _lib.IMPL_B, _lib.IMPL_C


def _torch():
    import torch
    return torch


class PackedWeight:
    """A weight prepacked for libfdpp: ``w`` is [N, ldw] (ldw = K rounded up to
    8, zero padded), the transpose of the reference's row-major B[K, N]."""

    __slots__ = ("w", "K", "N", "ldw")

    def __init__(self, w, K: int, N: int):
        self.w, self.K, self.N, self.ldw = w, int(K), int(N), int(w.stride(0))

    @property
    def dtype(self):
        return self.w.dtype

    @classmethod
    def from_nk(cls, w_nk):
        """Wrap an [N, K] (already K-major) weight, e.g. an nn.Linear weight."""
        torch = _torch()
        N, K = w_nk.shape
        if K % 8 or w_nk.stride(1) != 1 or w_nk.stride(0) % 8:
            w2 = torch.zeros((N, (K + 7) // 8 * 8), dtype=w_nk.dtype, device=w_nk.device)
            w2[:, :K] = w_nk
            w_nk = w2
        return cls(w_nk, K, N)


def pack_weight(b_kn, dtype=None, stream=None) -> PackedWeight:
    """Prepack the reference's B[K, N] on the device (fdpp_prepack_weight)."""
    torch = _torch()
    _lib.require_cuda()
    if not isinstance(b_kn, torch.Tensor):
        b_kn = torch.from_numpy(np.ascontiguousarray(b_kn, dtype=np.float32)).cuda()
    if dtype is None:
        dtype = b_kn.dtype if b_kn.dtype in (torch.float16, torch.bfloat16, torch.float32) else torch.float32
    b = b_kn.to(device="cuda", dtype=dtype).contiguous()
    if b.dim() != 2:
        raise ShapeError("weight must be 2-D [K, N]")
    K, N = b.shape
    ldw = (K + 7) // 8 * 8
    w = torch.empty((N, ldw), dtype=dtype, device=b.device)
    _lib.check(_lib.load().fdpp_prepack_weight(b.data_ptr(), w.data_ptr(), K, N, ldw,
                                               _lib.dtype_code(dtype), _lib.stream_handle(stream)),
               "prepack_weight")
    return PackedWeight(w, K, N)


_cache_lock = threading.Lock()
_pack_cache: dict = {}


def as_packed(b, dtype=None) -> PackedWeight:
    """PackedWeight for b (cached by tensor identity + version for CUDA tensors)."""
    torch = _torch()
    if isinstance(b, PackedWeight):
        return b
    if isinstance(b, torch.Tensor) and b.is_cuda:
        key = (b.data_ptr(), tuple(b.shape), tuple(b.stride()), b.dtype, b._version, dtype)
        with _cache_lock:
            hit = _pack_cache.get(key)
        if hit is not None:
            return hit
        pw = pack_weight(b, dtype)
        with _cache_lock:
            if len(_pack_cache) > 256:
                _pack_cache.clear()
            _pack_cache[key] = pw
        return pw
    return pack_weight(b, dtype)


def as_activation(a, dtype):
    """Device [M, K] activation with K padded to a multiple of 8."""
    torch = _torch()
    if not isinstance(a, torch.Tensor):
        a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    a = a.to(device="cuda", dtype=dtype)
    if a.dim() != 2:
        raise ShapeError("activation must be 2-D [M, K]")
    M, K = a.shape
    if K % 8 or a.stride(1) != 1 or a.stride(0) % 8 or a.data_ptr() % 16:
        a2 = torch.zeros((M, (K + 7) // 8 * 8), dtype=dtype, device=a.device)
        a2[:, :K] = a
        a = a2
    return a


def gemm_params(a, pw: PackedWeight, out, residual=None, block_x=0, ctas=0, stages=0):
    prm = _lib.GemmParams()
    prm.a, prm.lda = a.data_ptr(), a.stride(0)
    prm.w, prm.ldw = pw.w.data_ptr(), pw.ldw
    prm.c, prm.ldc = out.data_ptr(), out.stride(0)
    if residual is not None:
        prm.r, prm.ldr = residual.data_ptr(), residual.stride(0)
    prm.M, prm.N, prm.K = a.shape[0], pw.N, pw.ldw  # zero-padded K contributes exactly 0
    prm.dtype = _lib.dtype_code(a.dtype)
    prm.block_x, prm.ctas, prm.stages = int(block_x), int(ctas), int(stages)
    return prm


def run(impl: int, a, pw: PackedWeight, *, out=None, residual=None, block_x=0, ctas=0,
        stages=0, stream=None, ws_tag="gemm"):
    """Launch ImplA/B/C on device operands; returns out [M, N]."""
    torch = _torch()
    if a.shape[1] != pw.ldw:
        raise ShapeError(f"inner dims disagree: {tuple(a.shape)} x [K={pw.K}, N={pw.N}]")
    if a.dtype != pw.dtype:
        raise ValueError(f"activation dtype {a.dtype} != weight dtype {pw.dtype}")
    if out is None:
        out = torch.empty((a.shape[0], pw.N), dtype=a.dtype, device=a.device)
    prm = gemm_params(a, pw, out, residual, block_x, ctas, stages)
    lib = _lib.load()
    need = ctypes.c_size_t()
    _lib.check(lib.fdpp_gemm_workspace_size(impl, ctypes.byref(prm), ctypes.byref(need)), "gemm")
    if need.value:
        ws = workspace.get(need.value, a.device, tag=ws_tag, stream=stream)
        prm.workspace, prm.workspace_bytes = ws.data_ptr(), ws.numel()
    _lib.check(lib.fdpp_run_kernel(impl, ctypes.byref(prm), _lib.stream_handle(stream)),
               ("ImplA", "ImplB", "ImplC")[impl])
    return out


def plan(impl: int, M: int, N: int, K: int, *, block_x: int = 0, ctas: int = 0):
    """Host-only launch plan of ImplB (impl 1) / ImplC (impl 2) for an [M, K] x
    [N, K] problem (fdpp_gemm_plan): (CTAs, cluster split-K size or 0 for the
    persistent stream-K grid, token tile).  No device work."""
    prm = _lib.GemmParams()
    ld = (K + 7) // 8 * 8
    prm.lda, prm.ldw, prm.ldc = ld, ld, N
    prm.M, prm.N, prm.K = M, N, ld
    prm.dtype = _lib.F16
    prm.block_x, prm.ctas = block_x, ctas
    c, cl, bx = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.load().fdpp_gemm_plan(impl, ctypes.byref(prm), ctypes.byref(c), ctypes.byref(cl),
                                          ctypes.byref(bx)), "gemm_plan")
    return c.value, cl.value, bx.value


def reference_dtype(a):
    """Device dtype of a reference-signature call: fp16/bf16 tensors keep their
    dtype (tensor-core path); numpy arrays and float32 tensors compute in f32."""
    torch = _torch()
    if isinstance(a, torch.Tensor) and a.dtype in (torch.float16, torch.bfloat16):
        return a.dtype
    return torch.float32


def reference_call(impl: int, a, b, **kw):
    """Reference-signature call: a [M,K], b [K,N] (numpy f32 or tensors)."""
    torch = _torch()
    _lib.require_cuda()
    if a.shape[1] != (b.K if isinstance(b, PackedWeight) else b.shape[0]):
        raise ShapeError(f"inner dims disagree: {tuple(a.shape)} x {tuple(getattr(b, 'shape', (b.K, b.N)))}")
    was_numpy = not isinstance(a, torch.Tensor)
    dtype = reference_dtype(a)
    pw = as_packed(b, dtype)
    A = as_activation(a, dtype)
    if A.shape[1] != pw.ldw:
        raise ShapeError("inner dims disagree")
    c = run(impl, A, pw, **kw)
    return c.float().cpu().numpy() if was_numpy else c


def interleave_gate_up(pw: PackedWeight) -> PackedWeight:
    """Rows of a fused [gate; up] weight (N = 2F, F % 64 == 0) reordered so each
    128-row tile t holds gate rows [64t, 64t+64) then the matching up rows: the
    layout the SiLU*up epilogue (run_fused(silu_out=...)) consumes."""
    torch = _torch()
    F = pw.N // 2
    if pw.N % 128:
        raise ShapeError(f"gate|up width {pw.N} must be a multiple of 128")
    t = torch.arange(F // 64, device=pw.w.device)[:, None] * 64 + torch.arange(64, device=pw.w.device)[None, :]
    idx = torch.stack([t, t + F], 1).reshape(-1)
    return PackedWeight(pw.w[idx].contiguous(), pw.K, pw.N)


def permute_qkv_for_gemv(pw: PackedWeight) -> PackedWeight:
    """QKV rows per 128-row head reordered to [4j..4j+3, 64+4j..64+4j+3] per
    8-row block: each fused-GEMV CTA holds the RoPE pairs (i, i+64)."""
    torch = _torch()
    if pw.N % 128:
        raise ShapeError("QKV width must be (Hq + 2 Hkv) * 128")
    j = torch.arange(16, device=pw.w.device)[:, None] * 4 + torch.arange(4, device=pw.w.device)[None, :]
    head = torch.cat([j, j + 64], 1).reshape(-1)                       # 128 within-head rows
    idx = (torch.arange(pw.N // 128, device=pw.w.device)[:, None] * 128 + head[None, :]).reshape(-1)
    return PackedWeight(pw.w[idx].contiguous(), pw.K, pw.N)


def permute_gate_up_for_gemv(pw: PackedWeight) -> PackedWeight:
    """[gate; up] rows reordered to [gate 4c..4c+3, up 4c..4c+3] per 8-row block
    (the fused GEMV's SiLU*up epilogue)."""
    torch = _torch()
    F = pw.N // 2
    if F % 4:
        raise ShapeError("gate|up width must be a multiple of 8")
    c = torch.arange(F // 4, device=pw.w.device)[:, None] * 4 + torch.arange(4, device=pw.w.device)[None, :]
    idx = torch.cat([c, c + F], 1).reshape(-1)
    return PackedWeight(pw.w[idx].contiguous(), pw.K, pw.N)


def run_fused(a, pw: PackedWeight, *, out=None, residual=None, x_op: int = 0, ssq_in=None,
              ssq_tiles: int = 0, norm_w=None, eps: float = 1e-5, ssq_out=None, rope=None,
              silu_out=None, impl: str = "B", stream=None, ws_tag="gemm", allreduce=None,
              stages: int = 0):
    """ImplB with the decode-step fusions (fdpp_gemm_fused).

    x_op 1: the activation tile is RMSNorm(a) * norm_w, with the rows' sums of
    squares given as ssq_in[ssq_tiles, :] (written by the producer of ``a``).
    x_op 2: the activation is silu(a[:, :K]) * a[:, K:] (a = fused gate|up).
    ssq_out [N/128, M] (float32): per-128-column sums of squares of the stored
    output rows (for the next GEMM's x_op 1).  rope = dict(q_out, k_cache,
    v_cache, pos, theta): RoPE the q/k heads and append k/v at row pos[m]
    (QKV projection; ``out`` unused).  silu_out [M, N/2]: silu(gate) * up of a
    tile-interleaved gate|up weight (interleave_gate_up; ``out`` unused).
    impl "A": the GEMV form (fdpp_gemv_fused, M <= 2, x_op 0/3): ssq_out has
    N/8 tiles, rope / silu_out need the permute_*_for_gemv weight layouts.
    allreduce (a ``PeerAllReduce``, row-parallel projections): C becomes the sum
    of every rank's product plus ``residual`` once, exchanged inside the
    epilogue over peer memory (no separate collective)."""
    torch = _torch()
    K = pw.ldw
    if x_op == 2:
        if a.shape[1] < 2 * K:
            raise ShapeError("SiLU prologue needs a = [gate | up] with 2K columns")
    elif a.shape[1] != K:
        raise ShapeError(f"inner dims disagree: {tuple(a.shape)} x [K={pw.K}, N={pw.N}]")
    M = a.shape[0]
    if out is None and rope is None and silu_out is None:
        out = torch.empty((M, pw.N), dtype=a.dtype, device=a.device)
    prm = _lib.GemmParams()
    prm.a, prm.lda = a.data_ptr(), a.stride(0)
    prm.w, prm.ldw = pw.w.data_ptr(), pw.ldw
    if out is not None:
        prm.c, prm.ldc = out.data_ptr(), out.stride(0)
    if residual is not None:
        prm.r, prm.ldr = residual.data_ptr(), residual.stride(0)
    prm.M, prm.N, prm.K = M, pw.N, K
    prm.dtype = _lib.dtype_code(a.dtype)
    prm.stages = int(stages)
    fz = _lib.GemmFuse()
    fz.x_op = int(x_op)
    if x_op in (1, 3):
        fz.ssq_in, fz.ssq_tiles, fz.ssq_ld = ssq_in.data_ptr(), int(ssq_tiles), ssq_in.stride(0)
        fz.eps = float(eps)
    if x_op == 1:
        fz.norm_w = norm_w.data_ptr()
    if ssq_out is not None:
        fz.ssq_out, fz.ssq_out_ld = ssq_out.data_ptr(), ssq_out.stride(0)
    if rope is not None:
        kc = rope["k_cache"]
        fz.q_out, fz.k_cache, fz.v_cache = rope["q_out"].data_ptr(), kc.data_ptr(), rope["v_cache"].data_ptr()
        fz.pos = rope["pos"].data_ptr()
        fz.Hq, fz.Hkv = rope["q_out"].shape[1], kc.shape[1]
        fz.cache_stride_b, fz.cache_stride_h = kc.stride(0), kc.stride(1)
        fz.theta = float(rope.get("theta", 10000.0))
    if silu_out is not None:
        fz.act_out, fz.act_ld = silu_out.data_ptr(), silu_out.stride(0)
    if allreduce is not None:
        if impl == "A":
            raise ValueError("the fused all-reduce runs in the ImplB cluster epilogue")
        allreduce.fill(fz)
    lib = _lib.load()
    if impl == "A":
        _lib.check(lib.fdpp_gemv_fused(ctypes.byref(prm), ctypes.byref(fz), _lib.stream_handle(stream)),
                   "gemv_fused")
        return out
    need = ctypes.c_size_t()
    _lib.check(lib.fdpp_gemm_workspace_size(IMPL_B, ctypes.byref(prm), ctypes.byref(need)), "gemm_fused")
    if need.value:
        ws = workspace.get(need.value, a.device, tag=ws_tag, stream=stream)
        prm.workspace, prm.workspace_bytes = ws.data_ptr(), ws.numel()
    _lib.check(lib.fdpp_gemm_fused(ctypes.byref(prm), ctypes.byref(fz), _lib.stream_handle(stream)),
               "gemm_fused")
    return out
