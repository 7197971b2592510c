"""ctypes binding of libfdpp.so (include/fdpp.h).

This is the ONLY route to compute in the package: there is no CPU or
eager-PyTorch fallback.  If the library is missing or a CUDA device is absent,
every compute entry point raises instead of silently degrading.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FDPP_LIB") or os.path.join(_HERE, "_lib", "libfdpp.so")  # FDPP_LIB: dev override

F16, BF16, F32 = 0, 1, 2
ATTN_ASYNC, ATTN_SYNC = 0, 1
IMPL_A, IMPL_B, IMPL_C = 0, 1, 2

c_i32, c_i64, c_f32, c_vp, c_sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t


AR_MAX_WORLD = 8  # FDPP_AR_MAX_WORLD


class AttnParams(ctypes.Structure):
    """fdpp_attn_params (include/fdpp.h)."""
    _fields_ = [
        ("q", c_vp), ("k", c_vp), ("v", c_vp), ("o", c_vp),
        ("dtype", c_i32), ("B", c_i32), ("Hq", c_i32), ("Hkv", c_i32), ("L", c_i32), ("D", c_i32),
        ("q_stride_b", c_i64), ("q_stride_h", c_i64),
        ("kv_stride_b", c_i64), ("kv_stride_h", c_i64),
        ("o_stride_b", c_i64), ("o_stride_h", c_i64),
        ("seq_lens", c_vp),
        ("scale", c_f32), ("phi", c_f32), ("a", c_f32), ("b", c_f32),
        ("p", c_i32), ("splits_per_chunk", c_i32), ("mode", c_i32),
        ("row_flags", c_vp), ("viol_index", c_vp), ("rows_recomputed", c_vp),
        ("chunk_num", c_vp), ("chunk_den", c_vp),
        ("workspace", c_vp), ("workspace_bytes", c_sz),
        ("kv_prefetch", c_i32),
    ]


class GemmParams(ctypes.Structure):
    """fdpp_gemm_params (include/fdpp.h)."""
    _fields_ = [
        ("a", c_vp), ("lda", c_i64), ("w", c_vp), ("ldw", c_i64), ("c", c_vp), ("ldc", c_i64),
        ("r", c_vp), ("ldr", c_i64),
        ("M", c_i32), ("N", c_i32), ("K", c_i32), ("dtype", c_i32),
        ("block_x", c_i32), ("ctas", c_i32), ("stages", c_i32),
        ("workspace", c_vp), ("workspace_bytes", c_sz),
    ]


class GemmFuse(ctypes.Structure):
    """fdpp_gemm_fuse (include/fdpp.h)."""
    _fields_ = [
        ("x_op", c_i32), ("ssq_in", c_vp), ("ssq_tiles", c_i32), ("ssq_ld", c_i32),
        ("norm_w", c_vp), ("eps", c_f32), ("ssq_out", c_vp), ("ssq_out_ld", c_i32),
        ("q_out", c_vp), ("k_cache", c_vp), ("v_cache", c_vp), ("pos", c_vp),
        ("Hq", c_i32), ("Hkv", c_i32), ("cache_stride_b", c_i64), ("cache_stride_h", c_i64),
        ("theta", c_f32), ("act_out", c_vp), ("act_ld", c_i64),
        ("ar_rank", c_i32), ("ar_world", c_i32), ("ar_cap", c_i64), ("ar_ws", c_vp * AR_MAX_WORLD),
    ]


# name -> (restype, argtypes); must cover every function declared in include/fdpp.h
SIGNATURES = {
    "fdpp_last_error": (ctypes.c_char_p, []),
    "fdpp_version": (ctypes.c_int, []),
    "fdpp_sm_count": (ctypes.c_int, []),
    "fdpp_set_pdl": (ctypes.c_int, [ctypes.c_int]),
    "fdpp_attn_workspace_size": (c_i32, [ctypes.POINTER(AttnParams), ctypes.POINTER(c_sz)]),
    "fdpp_attn_plan": (c_i32, [ctypes.POINTER(AttnParams), ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)]),
    "fdpp_attn_launches": (c_i32, [ctypes.POINTER(AttnParams), ctypes.POINTER(c_i32)]),
    "fdpp_ar_workspace_size": (c_i32, [c_i32, c_i64, ctypes.POINTER(c_sz)]),
    "fdpp_ar_alloc": (c_i32, [c_sz, ctypes.POINTER(c_vp)]),
    "fdpp_ar_free": (c_i32, [c_vp]),
    "fdpp_ipc_get_handle": (c_i32, [c_vp, c_vp]),
    "fdpp_ipc_open": (c_i32, [c_vp, ctypes.POINTER(c_vp)]),
    "fdpp_ipc_close": (c_i32, [c_vp]),
    "fdpp_ar_check": (c_i32, [c_vp, ctypes.POINTER(c_i32)]),
    "fdpp_attn_decode": (c_i32, [ctypes.POINTER(AttnParams), c_vp]),
    "fdpp_prepack_weight": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i64, c_i32, c_vp]),
    "fdpp_gemm_workspace_size": (c_i32, [c_i32, ctypes.POINTER(GemmParams), ctypes.POINTER(c_sz)]),
    "fdpp_gemm_plan": (c_i32, [c_i32, ctypes.POINTER(GemmParams), ctypes.POINTER(c_i32), ctypes.POINTER(c_i32),
                               ctypes.POINTER(c_i32)]),
    "fdpp_impl_a_gemv": (c_i32, [ctypes.POINTER(GemmParams), c_vp]),
    "fdpp_impl_b_flat": (c_i32, [ctypes.POINTER(GemmParams), c_vp]),
    "fdpp_impl_c_gemm": (c_i32, [ctypes.POINTER(GemmParams), c_vp]),
    "fdpp_run_kernel": (c_i32, [c_i32, ctypes.POINTER(GemmParams), c_vp]),
    "fdpp_gemm_fused": (c_i32, [ctypes.POINTER(GemmParams), ctypes.POINTER(GemmFuse), c_vp]),
    "fdpp_gemv_fused": (c_i32, [ctypes.POINTER(GemmParams), ctypes.POINTER(GemmFuse), c_vp]),
    "fdpp_dispatch_choose": (c_i32, [c_i32, c_i32, c_i32]),
    "fdpp_first_sustained": (c_i32, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), c_i32, c_i32]),
    "fdpp_profile_decide": (c_i32, [ctypes.POINTER(c_i32), ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                    c_i32, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)]),
    "fdpp_chunk_bounds": (c_i32, [c_i64, c_i32, ctypes.POINTER(c_i64)]),
    "fdpp_rmsnorm": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_f32, c_i32, c_vp]),
    "fdpp_rope_append": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32,
                                 c_i64, c_i64, c_f32, c_i32, c_vp]),
    "fdpp_silu_mul": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "fdpp_embed": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_i32, c_vp]),
    "fdpp_row_ssq": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "fdpp_sample_logits": (c_i32, [ctypes.POINTER(AttnParams), c_i32, ctypes.c_uint64, c_vp, c_vp, c_vp]),
    "fdpp_softmax_reference": (c_i32, [c_vp, c_i32, c_vp, c_i32, c_vp]),
    "fdpp_softmax_unified": (c_i32, [c_vp, c_i32, c_f32, c_vp, c_vp, c_vp, c_vp]),
    "fdpp_softmax_overflow_index": (c_i32, [c_vp, c_i32, c_f32, c_vp, c_vp]),
    "fdpp_partial_softmax_sync": (c_i32, [c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "fdpp_argmax": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "fdpp_advance_positions": (c_i32, [c_vp, c_vp, c_i32, c_vp]),
}

_lib = None
_lock = threading.Lock()


class FdppError(RuntimeError):
    """CUDA / driver failure inside libfdpp."""


def load():
    """Load libfdpp.so (raises ImportError if it was never built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"libfdpp.so not found at {LIB_PATH}; run "
                    "`python -m paper_2311_01282_b200._build` (or __graft_entry__.build()). "
                    "There is no CPU fallback.")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int, what: str = ""):
    """Map an fdpp_status to the reference's exception types."""
    if status == 0:
        return
    msg = load().fdpp_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == 1:
        from .matrix import ShapeError
        raise ShapeError(text)
    if status in (2, 4, 5):
        raise ValueError(text)
    raise FdppError(text)


def require_cuda():
    """Fail loudly when no CUDA device is present (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2311_01282_b200 needs a CUDA (sm_100a) device; "
                           "there is no CPU fallback")
    load()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dtype_code(dt) -> int:
    import torch
    if dt == torch.float16:
        return F16
    if dt == torch.bfloat16:
        return BF16
    if dt == torch.float32:
        return F32
    raise ValueError(f"unsupported dtype {dt}")
