"""Decode-phase attention with asynchronized (unified-phi) softmax on B200
(reference: flatdecode/attention.py).

Drop-in surface: ``AttentionConfig`` (attention.py:46-56), ``AttnStats``
(:59-63), ``PartialAttnState`` (:30-43), ``attention_reference`` (:77-86),
``batch_decode_attention`` (:308-321), ``decode_attention_sync`` /
``decode_attention_async`` (:289-305) and ``async_chunk_state`` (:241-246),
plus ``async_partials`` (the chunk states of ``_async_partials``, :217-238).
These accept the reference's numpy f32 arrays (computed in fp32 on the
device, so inputs are bit-identical to the oracle's) or CUDA tensors.

B200 extension: ``decode_attention(q[B,Hq,D], k_cache[B,Hkv,L,D], v_cache,
cfg, mode)`` runs every head of a batch in one launch pair (GQA/MQA: query
head h reads kv head h // (Hq/Hkv)).  All compute goes through libfdpp's
``fdpp_attn_decode``; there is no CPU or eager fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

from . import _lib, workspace
from .matrix import ShapeError
from .softmax import ScalingCalibration

MODES = ("reference", "sync", "async")
_SUPPORTED_D = {2: (8, 16, 32, 64, 128, 256), 4: (4, 8, 16, 32, 64, 128)}


class PartialAttnState(NamedTuple):
    """One chunk's accumulation: num = sum e^(x-phi) v, den = sum e^(x-phi)."""

    num: np.ndarray
    den: np.float32
    overflow_index: int = -1

    @property
    def overflowed(self) -> bool:
        return self.overflow_index >= 0


AUTO = "auto"  # AttentionConfig.p: let the library plan the split for 148 SMs


@dataclass(frozen=True)
class AttentionConfig:
    """p = semantic split count (chunk_bounds(L, p)), validated like the
    reference (attention.py:46-56: an int >= 1, else ValueError); the B200
    extension ``p=AUTO`` ("auto", or ``AttentionConfig.auto(...)``) lets the
    library choose p for the machine.  splits_per_chunk = CTAs per chunk
    (0 = auto); it never changes results beyond fp32 summation order, and
    never changes flags."""

    p: object
    scale: float
    calib: Optional[ScalingCalibration] = None
    splits_per_chunk: int = 0

    def __post_init__(self):
        if self.p != AUTO:
            if isinstance(self.p, bool) or not isinstance(self.p, (int, np.integer)):
                raise ValueError(f"partition count must be an int >= 1 or {AUTO!r}, got {self.p!r}")
            if self.p < 1:
                raise ValueError(f"partition count must be >= 1, got {self.p}")
        if not self.scale > 0:
            raise ValueError(f"scale must be > 0, got {self.scale}")

    @classmethod
    def auto(cls, scale: float, calib: Optional[ScalingCalibration] = None, splits_per_chunk: int = 0):
        return cls(p=AUTO, scale=scale, calib=calib, splits_per_chunk=splits_per_chunk)

    @property
    def p_code(self) -> int:
        """The C ABI's p (0 = auto)."""
        return 0 if self.p == AUTO else int(self.p)


class AttnStats:
    """rows_recomputed / rescale_ops / max_ops with the reference's arithmetic
    (attention.py:154, :161, :284).  In async mode the count lives in a device
    counter and is read lazily (first attribute access synchronises), so the
    hot path never round-trips to the host.  ``row_mask`` is the per-row
    recompute flag set (the reference's ``redo``, attention.py:271)."""

    def __init__(self, rows_recomputed=0, rescale_ops=0, max_ops=0, *, _counter=None, _p=0,
                 _row_flags=None):
        self._rows = rows_recomputed
        self._rescale = rescale_ops
        self._max = max_ops
        self._counter = _counter
        self._p = _p
        self.row_flags = _row_flags

    def _resolve(self):
        if self._counter is not None:
            n = int(self._counter.item())
            self._counter = None
            self._rows += n
            self._rescale += 2 * n * self._p
            self._max += n * self._p + n

    @property
    def rows_recomputed(self) -> int:
        self._resolve()
        return self._rows

    @rows_recomputed.setter
    def rows_recomputed(self, v):
        self._resolve()
        self._rows = v

    @property
    def rescale_ops(self) -> int:
        self._resolve()
        return self._rescale

    @rescale_ops.setter
    def rescale_ops(self, v):
        self._resolve()
        self._rescale = v

    @property
    def max_ops(self) -> int:
        self._resolve()
        return self._max

    @max_ops.setter
    def max_ops(self, v):
        self._resolve()
        self._max = v

    @property
    def row_mask(self):
        return None if self.row_flags is None else self.row_flags.bool()

    def __repr__(self):
        return (f"AttnStats(rows_recomputed={self.rows_recomputed}, "
                f"rescale_ops={self.rescale_ops}, max_ops={self.max_ops})")


def _torch():
    import torch
    return torch


def plan(q, k_cache, cfg: AttentionConfig, L: Optional[int] = None, mode: str = "async"):
    """(p, splits_per_chunk) the library will use for these shapes in `mode`
    (the async launch may run the persistent kernel, whose auto p is 1)."""
    prm = _params(q, k_cache, k_cache, q, cfg, mode, L)
    c, s = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.load().fdpp_attn_plan(ctypes.byref(prm), ctypes.byref(c), ctypes.byref(s)), "attn_plan")
    return c.value, s.value


def launches(q, k_cache, cfg: AttentionConfig, L: Optional[int] = None, mode: str = "async") -> int:
    """Kernel launches one decode_attention call makes for these shapes: 1 when
    every row group is one cluster that recomputes its own flagged rows (the
    decode plans), else 2 (async + the flagged-list recompute launch)."""
    prm = _params(q, k_cache, k_cache, q, cfg, mode, L)
    n = ctypes.c_int32()
    _lib.check(_lib.load().fdpp_attn_launches(ctypes.byref(prm), ctypes.byref(n)), "attn_launches")
    return n.value


def _params(q, k, v, o, cfg, mode, L):
    B, Hq, D = q.shape
    Hkv = k.shape[1]
    if L is None:
        L = k.shape[2]
    prm = _lib.AttnParams()
    prm.q, prm.k, prm.v, prm.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr()
    prm.dtype = _lib.dtype_code(q.dtype)
    prm.B, prm.Hq, prm.Hkv, prm.L, prm.D = B, Hq, Hkv, int(L), D
    prm.q_stride_b, prm.q_stride_h = q.stride(0), q.stride(1)
    prm.kv_stride_b, prm.kv_stride_h = k.stride(0), k.stride(1)
    prm.o_stride_b, prm.o_stride_h = o.stride(0), o.stride(1)
    prm.scale = float(cfg.scale)
    if cfg.calib is not None:
        prm.phi, prm.a, prm.b = float(cfg.calib.phi), float(cfg.calib.a), float(cfg.calib.b)
    prm.p = cfg.p_code
    prm.splits_per_chunk = int(cfg.splits_per_chunk or 0)
    prm.mode = _lib.ATTN_ASYNC if mode == "async" else _lib.ATTN_SYNC
    return prm


def decode_attention(q, k_cache, v_cache, cfg: AttentionConfig, mode: str = "async", *,
                     out=None, L: Optional[int] = None, seq_lens=None, row_flags=None,
                     viol_index=None, chunk_num=None, chunk_den=None, counter=None, stream=None,
                     kv_prefetch: bool = False):
    """Batched decode attention on CUDA tensors.

    q [B, Hq, D]; k_cache / v_cache [B, Hkv, Lmax, D] (key rows contiguous);
    attends to the first L (default Lmax) keys, or to ``seq_lens[b]`` keys of
    batch row b when an int32 device tensor is given (read at run time).
    Returns (out [B, Hq, D], AttnStats).  Capturable into CUDA graphs when
    ``out`` / ``row_flags`` / ``counter`` are preallocated (no allocation, no
    host sync).  ``kv_prefetch``: the kernel launched just before wrote no K/V
    row except each batch row's last attended one (a decode step's append), so
    the rest may stream before the programmatic-dependent-launch wait.
    """
    torch = _torch()
    if mode not in ("sync", "async"):
        raise ValueError(f"mode must be one of ('sync', 'async') here, got {mode!r}")
    if mode == "async" and cfg.calib is None:
        raise ValueError("async mode requires a ScalingCalibration")
    if q.dim() != 3 or k_cache.dim() != 4 or v_cache.shape != k_cache.shape:
        raise ShapeError(f"expected q [B,Hq,D] and k/v [B,Hkv,L,D], got {tuple(q.shape)}, "
                         f"{tuple(k_cache.shape)}, {tuple(v_cache.shape)}")
    if q.shape[0] != k_cache.shape[0] or q.shape[2] != k_cache.shape[3]:
        raise ShapeError("batch / head dims of q and the cache disagree")
    if k_cache.stride(3) != 1 or k_cache.stride(2) != k_cache.shape[3] or q.stride(2) != 1:
        raise ShapeError("key rows must be contiguous ([..., L, D] row-major)")
    if v_cache.stride() != k_cache.stride():
        raise ShapeError("K and V caches must share strides")
    if not q.is_cuda:
        raise ValueError("decode_attention needs CUDA tensors (no CPU fallback)")
    B, Hq, D = q.shape
    if out is None:
        out = torch.empty((B, Hq, D), dtype=q.dtype, device=q.device)
    if row_flags is None:
        row_flags = torch.zeros((B, Hq), dtype=torch.uint8, device=q.device)
    if counter is None and mode == "async":
        counter = torch.zeros(1, dtype=torch.int32, device=q.device)
    prm = _params(q, k_cache, v_cache, out, cfg, mode, L)
    if seq_lens is not None:
        if seq_lens.dtype != torch.int32 or not seq_lens.is_cuda or seq_lens.numel() < B:
            raise ValueError("seq_lens must be an int32 CUDA tensor with one entry per batch row")
        prm.seq_lens = seq_lens.data_ptr()
    prm.row_flags = row_flags.data_ptr()
    prm.viol_index = viol_index.data_ptr() if viol_index is not None else None
    prm.rows_recomputed = counter.data_ptr() if counter is not None else None
    prm.chunk_num = chunk_num.data_ptr() if chunk_num is not None else None
    prm.chunk_den = chunk_den.data_ptr() if chunk_den is not None else None
    prm.kv_prefetch = 1 if kv_prefetch else 0
    lib = _lib.load()
    need = ctypes.c_size_t()
    _lib.check(lib.fdpp_attn_workspace_size(ctypes.byref(prm), ctypes.byref(need)), "attention")
    ws = workspace.get(need.value, q.device, tag="attn", stream=stream)
    prm.workspace, prm.workspace_bytes = ws.data_ptr(), ws.numel()
    c, s = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(lib.fdpp_attn_plan(ctypes.byref(prm), ctypes.byref(c), ctypes.byref(s)), "attention")
    _lib.check(lib.fdpp_attn_decode(ctypes.byref(prm), _lib.stream_handle(stream)), "attention")
    rows = B * Hq
    if mode == "sync":
        stats = AttnStats(0, 2 * rows * c.value, rows * c.value + rows)
    else:
        stats = AttnStats(_counter=counter, _p=c.value, _row_flags=row_flags)
    return out, stats


# ------------------------------------------------------------------ reference API

def _check_qkv(Q, K, V):
    if Q.ndim != 2 or K.ndim != 2 or V.ndim != 2:
        raise ShapeError("Q, K, V must be 2-D")
    if tuple(K.shape) != tuple(V.shape):
        raise ShapeError(f"K and V shapes disagree: {tuple(K.shape)} vs {tuple(V.shape)}")
    if Q.shape[1] != K.shape[1]:
        raise ShapeError(f"head dims disagree: Q {tuple(Q.shape)} vs K {tuple(K.shape)}")
    if K.shape[0] < 1:
        raise ShapeError("K/V cache must hold at least one row")


def _to_device(x, dtype=None):
    torch = _torch()
    _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.cuda()
        if dtype is not None:
            t = t.to(dtype)
        return t.contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _pad_d(t, D2):
    torch = _torch()
    if t.shape[-1] == D2:
        return t
    out = torch.zeros(t.shape[:-1] + (D2,), dtype=t.dtype, device=t.device)
    out[..., : t.shape[-1]] = t
    return out


def _single_head(Q, K, V, cfg, mode, *, want_partials=False):
    """The reference's one-head problem (M rows sharing one K/V) as a B=1,
    Hkv=1, Hq=M launch.  Returns (O [M, D] tensor, stats, extras)."""
    torch = _torch()
    was_numpy = not isinstance(Q, torch.Tensor)
    Qd, Kd, Vd = _to_device(Q), _to_device(K), _to_device(V)
    if Qd.dtype != Kd.dtype or Kd.dtype != Vd.dtype:
        Qd, Kd, Vd = Qd.float(), Kd.float(), Vd.float()
    _check_qkv(Qd, Kd, Vd)
    M, D = Qd.shape
    L = Kd.shape[0]
    esz = Qd.element_size()
    D2 = next((d for d in _SUPPORTED_D[esz] if d >= D), None)
    if D2 is None:
        raise ValueError(f"head dim {D} not supported for {Qd.dtype}")
    q = _pad_d(Qd, D2).reshape(1, M, D2)
    k = _pad_d(Kd, D2).reshape(1, 1, L, D2)
    v = _pad_d(Vd, D2).reshape(1, 1, L, D2)
    extras = {}
    kw = {}
    if want_partials:
        p = int(cfg.p)
        extras["viol"] = kw["viol_index"] = torch.full((1, M, p), -1, dtype=torch.int32, device=q.device)
        extras["num"] = kw["chunk_num"] = torch.zeros((1, M, p, D2), dtype=torch.float32, device=q.device)
        extras["den"] = kw["chunk_den"] = torch.zeros((1, M, p), dtype=torch.float32, device=q.device)
    o, stats = decode_attention(q, k, v, cfg, mode, **kw)
    o = o[0, :, :D]
    if "num" in extras:
        extras["num"] = extras["num"][0, :, :, :D]
        extras["den"] = extras["den"][0]
        extras["viol"] = extras["viol"][0]
    if stats.row_flags is not None:
        stats.row_flags = stats.row_flags[0]
    return o, stats, extras, was_numpy


def attention_reference(Q, K, V, scale):
    """softmax(scale Q K^T) V with every intermediate in float64, on the device."""
    torch = _torch()
    was_numpy = not isinstance(Q, torch.Tensor)
    Qd, Kd, Vd = _to_device(Q), _to_device(K), _to_device(V)
    _check_qkv(Qd, Kd, Vd)
    from .reference_ops import attention_f64
    out = attention_f64(Qd, Kd, Vd, float(scale))
    return out.cpu().numpy() if was_numpy else out


def batch_decode_attention(Q, K, V, cfg: AttentionConfig, mode: str):
    """Apply the selected kernel to every query row (attention.py:308-321).

    Returns (O, AttnStats); O is float32 numpy for numpy inputs, else a tensor
    of the input dtype.  In async mode the counters reflect only the work of
    the recomputed rows; ``stats.row_mask`` is the recompute flag set."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    if mode == "reference":
        return attention_reference(Q, K, V, cfg.scale), AttnStats()
    if mode == "async" and cfg.calib is None:
        raise ValueError("async mode requires a ScalingCalibration")
    o, stats, _, was_numpy = _single_head(Q, K, V, cfg, mode)
    if was_numpy:
        o = o.float().cpu().numpy()
        if stats.row_flags is not None:
            stats.row_flags = stats.row_flags.cpu()
    return o, stats


def decode_attention_sync(q, K, V, cfg: AttentionConfig):
    """Synchronized split-cache attention for one query row (attention.py:289-294)."""
    o, _ = batch_decode_attention(_row(q), K, V, cfg, "sync")
    return o[0]


def decode_attention_async(q, K, V, cfg: AttentionConfig):
    """Unified-scaling attention for one query row; returns (o, recomputed)."""
    o, stats = batch_decode_attention(_row(q), K, V, cfg, "async")
    return o[0], stats.rows_recomputed > 0


def _row(q):
    torch = _torch()
    if isinstance(q, torch.Tensor):
        return q.reshape(1, -1)
    return np.reshape(q, (1, -1))


def async_partials(Q, K, V, cfg: AttentionConfig):
    """Chunk states of the async kernel: (num [M,p,D] f32, den [M,p] f32,
    viol [M,p] int64) with the reference's conventions (attention.py:217-238):
    a violating chunk is zeroed and reports its first out-of-band key; a chunk
    whose state is not f32-representable reports its lower bound."""
    if cfg.calib is None:
        raise ValueError("async mode requires a ScalingCalibration")
    if cfg.p == AUTO:
        raise ValueError("async_partials needs an explicit p")
    _, _, ex, _ = _single_head(Q, K, V, cfg, "async", want_partials=True)
    return (ex["num"].cpu().numpy(), ex["den"].cpu().numpy(),
            ex["viol"].cpu().numpy().astype(np.int64))


def async_chunk_state(q, K, V, lo: int, hi: int, cfg: AttentionConfig) -> PartialAttnState:
    """One chunk's state for K/V rows [lo, hi) of a single query row (attention.py:241-246)."""
    torch = _torch()
    Kc = K[lo:hi] if isinstance(K, (np.ndarray, torch.Tensor)) else np.asarray(K)[lo:hi]
    Vc = V[lo:hi] if isinstance(V, (np.ndarray, torch.Tensor)) else np.asarray(V)[lo:hi]
    one = AttentionConfig(p=1, scale=cfg.scale, calib=cfg.calib)
    num, den, viol = async_partials(_row(q), Kc, Vc, one)
    v = int(viol[0, 0])
    return PartialAttnState(num[0, 0], np.float32(den[0, 0]), v + lo if v >= 0 else -1)


def sample_logits(q, k_cache, scale: float, n: int, *, seq_lens=None, seed: int = 0,
                  return_index: bool = False):
    """Calibration producer: ``n`` logits
    ``scale * q[b, h] . k[b, h // G, key]`` at pseudo-random (b, h, key < seq_lens[b])
    computed on the device (``fdpp_sample_logits``) -- the sample the
    reference's ``calibrate`` (softmax.py:219-266) fits phi and the band to.
    Returns a float32 CUDA tensor (and the [n, 3] int32 (b, h, key) indices)."""
    torch = _torch()
    _lib.require_cuda()
    if n < 1:
        raise ValueError("n must be >= 1")
    prm = _params(q, k_cache, k_cache, q, AttentionConfig.auto(scale), "sync", None)
    if seq_lens is not None:
        if seq_lens.dtype != torch.int32 or not seq_lens.is_cuda:
            raise ValueError("seq_lens must be an int32 CUDA tensor")
        prm.seq_lens = seq_lens.data_ptr()
    out = torch.empty(n, dtype=torch.float32, device=q.device)
    idx = torch.empty((n, 3), dtype=torch.int32, device=q.device) if return_index else None
    _lib.check(_lib.load().fdpp_sample_logits(ctypes.byref(prm), int(n), int(seed) & (2 ** 64 - 1),
                                              out.data_ptr(), idx.data_ptr() if idx is not None else None,
                                              _lib.stream_handle()), "sample_logits")
    return (out, idx) if return_index else out
