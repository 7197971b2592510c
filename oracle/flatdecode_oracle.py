"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference package ``flatdecode``
(/root/reference/pkg/src/flatdecode) used to check the B200 product path.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; the product package (``paper_2311_01282_b200``) never
does, and it fails loudly when its CUDA library is missing instead of falling
back here.

Pinned against the reference itself: ``tests/golden/make_golden.py`` ran the
real reference in the build container and committed its outputs as
``tests/golden/*.npz|json``; ``tests/test_oracle_golden.py`` checks every
function below against them.

Heavy loops live in ``ref_kernels.c`` (a plain-C restatement of the numba
kernels, built by ``oracle/Makefile``); this module restates the host-side
logic around them.  Every function cites the reference file:line it follows.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libref_kernels.so")

# softmax.py:16-19
EXP_OVERFLOW_BOUND = 88.0
EXP_UNDERFLOW_BOUND = -87.0

# dispatch.py:24-27
DEFAULT_M_SWEEP = (1, 2, 4, 8, 16, 32, 64, 128, 256)
GEMV_PANEL = 256
BLOCK_MNK = 64
TABLE_MAGIC = "flatdecode-dispatch"
TABLE_VERSION = "v1"
KERNEL_NAMES = ("ImplA", "ImplB", "ImplC")  # dispatch.py:36-39

# flatgemm.py:18-20
MICROKERNEL_ROWS = 8
MICROKERNEL_WIDTH = 8
DEFAULT_B_K = 32


# --------------------------------------------------------------------------- C library

def build_lib(force: bool = False) -> str:
    """Compile ref_kernels.c (gcc, pthreads) into oracle/build/."""
    src = os.path.join(_HERE, "ref_kernels.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "build/libref_kernels.so"], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = ctypes.CDLL(_LIB_PATH)
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        i64 = ctypes.c_int64
        f32 = ctypes.c_float
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_set_threads.restype = ctypes.c_int
        L.oracle_async_partials.argtypes = [f32p, f32p, f32p, i64, i64, f32, f32, f32, f32,
                                            i64p, i64, f64p, f64p, i64p]
        L.oracle_sync_partials.argtypes = [f32p, f32p, f32p, i64, i64, f32, i64p, i64,
                                           f32p, f32p, f32p]
        L.oracle_gemm_f64.argtypes = [f32p, f32p, f32p, i64, i64, i64]
        L.oracle_gemv_rows.argtypes = [f32p, f32p, f32p, i64, i64, i64, i64]
        L.oracle_flat_gemm.argtypes = [f32p, f32p, f32p, i64, i64, i64, i64, i64, ctypes.c_int]
        L.oracle_blocked_gemm.argtypes = [f32p, f32p, f32p, i64, i64, i64, i64, i64, i64]
        for fn in ("oracle_async_partials", "oracle_sync_partials", "oracle_gemm_f64",
                   "oracle_gemv_rows", "oracle_flat_gemm", "oracle_blocked_gemm"):
            getattr(L, fn).restype = None
        _lib = L
    return _lib


def set_threads(n: int) -> int:
    return lib().oracle_set_threads(int(n))


def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


# --------------------------------------------------------------------------- softmax.py

@dataclass(frozen=True)
class Calib:
    """softmax.py:175-197 (ScalingCalibration) — phi plus the open band (a, b)."""
    phi: float
    a: float
    b: float
    coverage: float = 1.0

    def __post_init__(self):
        if not self.a < self.b:
            raise ValueError("need a < b")
        if self.b >= EXP_OVERFLOW_BOUND or self.a <= EXP_UNDERFLOW_BOUND:
            raise ValueError("band breaks the f32 exponent budget")
        if not 0.0 <= self.coverage <= 1.0:
            raise ValueError("coverage out of range")


def chunk_bounds(n: int, p: int) -> np.ndarray:
    """softmax.py:103-110."""
    if not 1 <= p <= n:
        raise ValueError(f"partition count must be in [1, {n}], got {p}")
    base = n // p
    bounds = np.arange(p + 1, dtype=np.int64) * base
    bounds[p] = n
    return bounds


def check_bounds(x, calib) -> Optional[int]:
    """softmax.py:200-210: first index with x-phi outside the open band."""
    x = np.asarray(x, dtype=np.float32)
    t = x - np.float32(calib.phi)
    viol = (t <= np.float32(calib.a)) | (t >= np.float32(calib.b))
    idx = np.nonzero(viol)[0]
    return int(idx[0]) if idx.size else None


def softmax_reference_f64(x) -> np.ndarray:
    """softmax.py:90-94."""
    x = np.asarray(x, dtype=np.float64)
    e = np.exp(x - x.max())
    return e / e.sum()


def softmax_unified(x, phi) -> np.ndarray:
    """softmax.py:146-172 (returns None-free result; raises like the reference)."""
    x = _f32(x)
    with np.errstate(over="ignore", under="ignore"):
        e = np.exp(x - np.float32(phi))
    bad = np.nonzero(~np.isfinite(e))[0]
    if bad.size:
        raise OverflowError(int(bad[0]))
    total = e.sum(dtype=np.float64)
    if total == 0.0:
        raise ZeroDivisionError("all scaled exponentials underflowed")
    return (e / total).astype(np.float32)


def _counted_coverage(samples, phi, a, b) -> float:
    """softmax.py:213-216."""
    t = samples - np.float32(phi)
    inside = (t > np.float32(a)) & (t < np.float32(b))
    return float(inside.sum()) / samples.size


def calibrate(samples, target_coverage: float, margin: float = 1.0) -> Calib:
    """softmax.py:219-266 (quantile anchor, widening loop, f32 rounding)."""
    samples = np.ascontiguousarray(samples, dtype=np.float32).ravel()
    if samples.size == 0:
        raise ValueError("samples must be non-empty")
    if not 0.5 < target_coverage <= 1.0:
        raise ValueError("target_coverage must be in (0.5, 1]")
    if not 0.0 < margin < -EXP_UNDERFLOW_BOUND:
        raise ValueError("bad margin")
    s = np.sort(samples.astype(np.float64))
    n = s.size
    q_lo = (1.0 - target_coverage) / 2.0
    q_hi = 1.0 - q_lo
    phi = float(np.quantile(s, q_lo, method="linear"))
    hi = float(np.quantile(s, q_hi, method="linear"))
    a = -float(margin)
    b = (hi - phi) + float(margin)
    lo_i = int(np.searchsorted(s, phi, side="left"))
    hi_i = int(np.searchsorted(s, hi, side="right")) - 1
    while _counted_coverage(samples, phi, a, b) < target_coverage:
        if lo_i == 0 and hi_i == n - 1 and phi <= s[0] and hi >= s[-1]:
            break
        lo_i = max(0, lo_i - 1)
        hi_i = min(n - 1, hi_i + 1)
        phi = min(phi, float(s[lo_i]))
        hi = max(hi, float(s[hi_i]))
        b = (hi - phi) + float(margin)
    if float(np.float32(b)) >= EXP_OVERFLOW_BOUND:
        raise ArithmeticError("uncalibratable range")
    coverage = _counted_coverage(samples, phi, a, b)
    return Calib(phi=float(np.float32(phi)), a=float(np.float32(a)),
                 b=float(np.float32(b)), coverage=coverage)


# --------------------------------------------------------------------------- attention.py

def attention_reference(Q, K, V, scale) -> np.ndarray:
    """attention.py:77-86: softmax(scale*QK^T)V in f64, rounded to f32."""
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    S = float(scale) * (Q.astype(np.float64) @ K.astype(np.float64).T)
    E = np.exp(S - S.max(axis=1, keepdims=True))
    P = E / E.sum(axis=1, keepdims=True)
    return (P @ V.astype(np.float64)).astype(np.float32)


def async_partials(Q, K, V, scale, calib, bounds):
    """attention.py:217-238: chunk partials + f32 rounding + 'unrepresentable
    state => violation at chunk lo'.  Returns (num32[M,p,d], den32[M,p], viol[M,p])."""
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    M, d = Q.shape
    p = bounds.size - 1
    num = np.empty((M, p, d), dtype=np.float64)
    den = np.empty((M, p), dtype=np.float64)
    viol = np.empty((M, p), dtype=np.int64)
    lib().oracle_async_partials(Q, K, V, M, d, np.float32(scale), np.float32(calib.phi),
                                np.float32(calib.a), np.float32(calib.b), bounds, p,
                                num, den, viol)
    num32 = num.astype(np.float32)
    den32 = den.astype(np.float32)
    unrep = ~(np.isfinite(den32) & np.isfinite(num32).all(axis=2))
    if unrep.any():
        viol = viol.copy()
        viol[unrep & (viol < 0)] = bounds[:-1][np.nonzero(unrep & (viol < 0))[1]]
    return num32, den32, viol


def sync_partials(Q, K, V, scale, bounds):
    """attention.py:89-120."""
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    M, d = Q.shape
    p = bounds.size - 1
    m = np.empty((M, p), dtype=np.float32)
    l = np.empty((M, p), dtype=np.float32)
    acc = np.empty((M, p, d), dtype=np.float32)
    lib().oracle_sync_partials(Q, K, V, M, d, np.float32(scale), bounds, p, m, l, acc)
    return m, l, acc


def sync_join(m, l, acc, stats: dict):
    """attention.py:149-162: Eq. (2) merge in chunk order, f32; counts ops."""
    M, p = m.shape
    m_row = m.max(axis=1)
    stats["max_ops"] += M * p + M
    num = np.zeros((M, acc.shape[2]), dtype=np.float32)
    den = np.zeros(M, dtype=np.float32)
    for j in range(p):
        f = np.exp(m[:, j] - m_row)
        num += f[:, None] * acc[:, j, :]
        den += f * l[:, j]
        stats["rescale_ops"] += 2 * M
    return num / den[:, None]


def _new_stats():
    return {"rows_recomputed": 0, "rescale_ops": 0, "max_ops": 0}


def batch_sync(Q, K, V, p, scale, stats):
    """attention.py:257-263."""
    bounds = chunk_bounds(np.asarray(K).shape[0], p)
    m, l, acc = sync_partials(Q, K, V, scale, bounds)
    return sync_join(m, l, acc, stats)


def batch_async(Q, K, V, p, scale, calib, stats):
    """attention.py:266-286.  Also returns the per-row recompute mask (redo)."""
    Q = _f32(Q)
    bounds = chunk_bounds(np.asarray(K).shape[0], p)
    num, den, viol = async_partials(Q, K, V, scale, calib, bounds)
    redo = (viol >= 0).any(axis=1)
    M, pp, d = num.shape
    out = np.empty((M, d), dtype=np.float32)
    ok = ~redo
    if ok.any():
        num_row = np.zeros((int(ok.sum()), d), dtype=np.float64)
        den_row = np.zeros(int(ok.sum()), dtype=np.float64)
        for j in range(pp):
            num_row += num[ok, j, :]
            den_row += den[ok, j]
        out[ok] = (num_row / den_row[:, None]).astype(np.float32)
    if redo.any():
        stats["rows_recomputed"] += int(redo.sum())
        out[redo] = batch_sync(Q[redo], K, V, p, scale, stats)
    return out, redo


def batch_decode_attention(Q, K, V, p, scale, calib, mode):
    """attention.py:308-321.  Returns (O, stats dict, redo mask or None)."""
    stats = _new_stats()
    if mode == "reference":
        return attention_reference(Q, K, V, scale), stats, None
    if mode == "sync":
        return batch_sync(Q, K, V, p, scale, stats), stats, None
    if mode == "async":
        out, redo = batch_async(Q, K, V, p, scale, calib, stats)
        return out, stats, redo
    raise ValueError(mode)


def row_guard_ok(Q, K, scale, calib, delta: float = 1e-3):
    """Per-row robustness of the band decision under accumulation-order changes
    (SURVEY §7.4 item 3): a row is 'clearly in' if every shifted logit is at
    least delta inside the band and 'clearly out' if one is at least delta
    outside.  Returns (clear_mask, outside_mask) in f64."""
    t = float(scale) * (np.asarray(Q, np.float64) @ np.asarray(K, np.float64).T) - float(calib.phi)
    inside = ((t > calib.a + delta) & (t < calib.b - delta)).all(axis=1)
    outside = ((t <= calib.a - delta) | (t >= calib.b + delta)).any(axis=1)
    return inside | outside, outside


# --------------------------------------------------------------------------- matrix.py / GEMMs

def pad_rows(a, multiple: int):
    """matrix.py:53-67."""
    if multiple < 1:
        raise ValueError("padding multiple must be >= 1")
    rows = a.shape[0]
    padded = ((rows + multiple - 1) // multiple) * multiple
    if padded == rows:
        return a
    out = np.zeros((padded, a.shape[1]), dtype=np.float32)
    out[:rows] = a
    return out


def gemm_oracle(a, b) -> np.ndarray:
    """matrix.py:90-104: f64 ascending-k accumulation, rounded to f32."""
    a, b = _f32(a), _f32(b)
    c = np.empty((a.shape[0], b.shape[1]), dtype=np.float32)
    lib().oracle_gemm_f64(a, b, c, a.shape[0], b.shape[1], a.shape[1])
    return c


def impl_a_gemv(a, b) -> np.ndarray:
    """dispatch.py:73-90 (ImplA)."""
    a, b = _f32(a), _f32(b)
    c = np.empty((a.shape[0], b.shape[1]), dtype=np.float32)
    lib().oracle_gemv_rows(a, b, c, a.shape[0], a.shape[1], b.shape[1], GEMV_PANEL)
    return c


def flat_gemm(a, b, b_n: int, b_k: int, m_pad: int = MICROKERNEL_ROWS,
              double_buffer: bool = False) -> np.ndarray:
    """flatgemm.py:215-242 (ImplB kernel with an explicit tile)."""
    a, b = _f32(a), _f32(b)
    M, N, K = a.shape[0], b.shape[1], b.shape[0]
    bn, bk = min(b_n, N), min(b_k, K)
    A = _f32(pad_rows(a, m_pad))
    C = np.zeros((A.shape[0], N), dtype=np.float32)
    lib().oracle_flat_gemm(A, b, C, A.shape[0], K, N, bn, bk, int(double_buffer))
    return C[:M]


def impl_b_flat(a, b, workers: int) -> np.ndarray:
    """dispatch.py:140-145 (ImplB under select_tile)."""
    a = np.asarray(a)
    t = select_tile(a.shape[0], np.asarray(b).shape[1], np.asarray(b).shape[0], workers)
    return flat_gemm(a, b, t["b_n"], t["b_k"], t["m_pad"], t["double_buffer"])


def impl_c_blocked(a, b) -> np.ndarray:
    """dispatch.py:117-137 (ImplC)."""
    a, b = _f32(a), _f32(b)
    c = np.zeros((a.shape[0], b.shape[1]), dtype=np.float32)
    lib().oracle_blocked_gemm(a, b, c, a.shape[0], a.shape[1], b.shape[1],
                              BLOCK_MNK, BLOCK_MNK, BLOCK_MNK)
    return c


# --------------------------------------------------------------------------- flatgemm.py host logic

def arithmetic_intensity(m, n, k, b_n, b_k):
    """flatgemm.py:49-69 -> (flops, traffic_elements, intensity, parallelism)."""
    if min(m, n, k) < 1:
        raise ValueError("dims")
    if not (1 <= b_n <= n and 1 <= b_k <= k):
        raise ValueError("tile")
    flops = 2 * m * n * k
    n_tiles = (n * k) / (b_n * b_k)
    traffic = (m * b_k + b_n * b_k) * n_tiles + m * n
    return flops, traffic, flops / traffic, n / b_n


def _width_candidates(n):
    """flatgemm.py:72-75."""
    c = [w for w in (1, 2, 4) if w <= n]
    c += list(range(MICROKERNEL_WIDTH, n + 1, MICROKERNEL_WIDTH))
    return c


def select_tile(m, n, k, workers, parallel_target=None):
    """flatgemm.py:78-102."""
    if min(m, n, k) < 1:
        raise ValueError("dims")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if parallel_target is None:
        parallel_target = 4 * workers
    b_k = min(DEFAULT_B_K, k)
    cands = _width_candidates(n)
    if n <= parallel_target * MICROKERNEL_WIDTH:
        feasible = [w for w in cands if n / w >= workers] or cands
        b_n = min(feasible, key=lambda w: (abs(n / w - parallel_target), w))
        return {"b_n": b_n, "b_k": b_k, "m_pad": MICROKERNEL_ROWS, "double_buffer": False}
    feasible = [w for w in cands if n / w >= workers]
    return {"b_n": max(feasible), "b_k": b_k, "m_pad": MICROKERNEL_ROWS, "double_buffer": True}


def double_buffer_pipeline(n_k_tiles: int):
    """flatgemm.py:107-126."""
    if n_k_tiles < 1:
        raise ValueError("need at least one K tile")
    ev = [("fill", 0, 0)]
    if n_k_tiles > 1:
        ev.append(("fill", 1, 1))
    for t in range(n_k_tiles):
        ev.append(("compute", t, t % 2))
        if t + 2 < n_k_tiles:
            ev.append(("fill", t + 2, (t + 2) % 2))
    return ev


# --------------------------------------------------------------------------- dispatch.py host logic

def dispatch(m, m1, m2) -> str:
    """dispatch.py:189-197 on one (m1, m2) entry."""
    if m < m1:
        return "ImplA"
    if m < m2:
        return "ImplB"
    return "ImplC"


def first_sustained(costs_new, costs_old, start=0):
    """dispatch.py:248-265."""
    n = len(costs_new)
    for i in range(start, n):
        if costs_new[i] > costs_old[i]:
            continue
        if i < n - 1 and costs_new[i + 1] > costs_old[i + 1]:
            continue
        relapsed = any(costs_new[j] > costs_old[j] and costs_new[j + 1] > costs_old[j + 1]
                       for j in range(i + 1, n - 1))
        if not relapsed:
            return i
    return None


def decide(m_sweep, med_a, med_b, med_c):
    """dispatch.py:327-338: inflection points from per-M medians -> (m1, m2)."""
    beyond = 2 * m_sweep[-1]
    i1 = first_sustained(med_b, med_a)
    if i1 is None:
        iac = first_sustained(med_c, med_a)
        m1 = m2 = m_sweep[iac] if iac is not None else beyond
    else:
        i2 = first_sustained(med_c, med_b, start=i1)
        m1 = m_sweep[i1]
        m2 = max(m1, m_sweep[i2]) if i2 is not None else beyond
    return m1, m2


def median_mad(samples):
    """timing.py:8-13."""
    s = np.asarray(samples, dtype=np.float64)
    med = float(np.median(s))
    return med, float(np.median(np.abs(s - med)))


def table_text(fingerprint: str, entries) -> str:
    """dispatch.py:206-211: header + sorted 'N K M1 M2' lines."""
    lines = [f"{TABLE_MAGIC} {TABLE_VERSION} {fingerprint}"]
    for (n, k) in sorted(entries):
        m1, m2 = entries[(n, k)]
        lines.append(f"{n} {k} {m1} {m2}")
    return "\n".join(lines) + "\n"


# --------------------------------------------------------------------------- metrics.py

def rel_error_elementwise(actual, oracle, floor: float = 1e-12) -> float:
    """metrics.py:12-16."""
    a = np.asarray(actual, dtype=np.float64)
    o = np.asarray(oracle, dtype=np.float64)
    return float((np.abs(a - o) / np.maximum(np.abs(o), floor)).max())


def rel_error_rowwise(actual, oracle, floor: float = 1e-8) -> float:
    """metrics.py:19-32."""
    a = np.asarray(actual, dtype=np.float64)
    o = np.asarray(oracle, dtype=np.float64)
    if a.ndim == 1:
        a, o = a[None, :], o[None, :]
    diff = np.abs(a - o).max(axis=1)
    scale = np.maximum(np.abs(o).max(axis=1), floor)
    return float((diff / scale).max())
