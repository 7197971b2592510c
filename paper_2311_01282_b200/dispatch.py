"""Heuristic dataflow dispatch on B200 (reference: flatdecode/dispatch.py).

Three device implementations behind the reference's names:

  ImplA  impl_a_gemv     CUDA-core GEMV (M <= 8), weights streamed once
  ImplB  impl_b_flat     swap-AB tcgen05 flat GEMM (tokens on the MMA N axis)
  ImplC  impl_c_blocked  conventional tcgen05 GEMM (tokens on the MMA M axis)

The offline decision flow (``profile_shape``, dispatch.py:278-338) measures
the three kernels with CUDA events (L2 flushed before every rep, median of
reps, the 20%-MAD stability gate) over an ascending M sweep and locates the
per-[N, K] inflection points M1 (ImplB overtakes ImplA) and M2 (ImplC
overtakes ImplB).  ``_first_sustained`` and the final decision run natively in
libfdpp (fdpp_first_sustained / fdpp_profile_decide) so a C/Go caller makes
bit-identical choices.  Tables persist in the reference's text format
(``flatdecode-dispatch v1 <fingerprint>``, dispatch.py:206-243) with a B200
fingerprint.  ImplA is GEMV-only: above M = 8 its measured cost is +inf, so
the flow never selects it there.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from . import gemm as _g
from .matrix import GemmShape, ShapeError
from .timing import measure, median_mad

DEFAULT_M_SWEEP = (1, 2, 4, 8, 16, 32, 64, 128, 256)
# the reference's sweep (dispatch.py:24) with one extra point between the flat
# band and the 128-token conventional tile, where ImplB starts re-streaming
# weights per 64-token tile
B200_M_SWEEP = (1, 2, 4, 8, 16, 32, 64, 96, 128, 256)
DEFAULT_REPS = 7
DEFAULT_WARMUP = 2
GEMV_MAX_M = 8

TABLE_MAGIC = "flatdecode-dispatch"
TABLE_VERSION = "v1"


class KernelChoice(Enum):
    IMPL_A = "ImplA"
    IMPL_B = "ImplB"
    IMPL_C = "ImplC"


_CODE = {KernelChoice.IMPL_A: _lib.IMPL_A, KernelChoice.IMPL_B: _lib.IMPL_B,
         KernelChoice.IMPL_C: _lib.IMPL_C}
_FROM_CODE = {v: k for k, v in _CODE.items()}


class UnknownShape(KeyError):
    def __init__(self, n, k):
        self.n = n
        self.k = k
        super().__init__(f"no dispatch entry for [N={n}, K={k}]")


class TimingUnstable(RuntimeError):
    pass


# ----------------------------------------------------------------- implementations

def impl_a_gemv(a, b, **kw):
    """ImplA: CUDA-core GEMV for M <= 8 (dispatch.py:73-90); larger M runs in
    8-row slabs (each slab streams the weights once)."""
    if a.shape[1] != (b.K if isinstance(b, _g.PackedWeight) else b.shape[0]):
        raise ShapeError(f"inner dims disagree: {tuple(a.shape)} x {tuple(getattr(b, 'shape', ()))}")
    M = a.shape[0]
    if M <= GEMV_MAX_M or _g.reference_dtype(a) == _torch_f32():
        return _g.reference_call(_g.IMPL_A, a, b, **kw)
    pw = _g.as_packed(b, _dtype_of(a))
    parts = [_g.reference_call(_g.IMPL_A, a[i:i + GEMV_MAX_M], pw) for i in range(0, M, GEMV_MAX_M)]
    if isinstance(parts[0], np.ndarray):
        return np.concatenate(parts)
    import torch
    return torch.cat(parts)


def _dtype_of(a):
    return _g.reference_dtype(a)


def _torch_f32():
    import torch
    return torch.float32


def impl_b_flat(a, b, workers: int = None, **kw):
    """ImplB: the flat GEMM under its device tile heuristic (dispatch.py:140-145).
    ``workers`` is accepted for API compatibility (the device uses 148 SMs)."""
    return _g.reference_call(_g.IMPL_B, a, b, **kw)


def impl_c_blocked(a, b, **kw):
    """ImplC: conventional tcgen05 GEMM, 128-row token tiles (dispatch.py:117-137)."""
    return _g.reference_call(_g.IMPL_C, a, b, **kw)


IMPLEMENTATIONS = {
    KernelChoice.IMPL_A: impl_a_gemv,
    KernelChoice.IMPL_B: impl_b_flat,
    KernelChoice.IMPL_C: impl_c_blocked,
}


def run_kernel(choice: KernelChoice, a, b):
    return IMPLEMENTATIONS[choice](a, b)


def run_device(choice: KernelChoice, a, pw, *, out=None, residual=None, stream=None, **kw):
    """Hot-path launch on device operands (no conversion, no allocation when
    ``out`` is given): what the decode step and the bench call."""
    return _g.run(_CODE[choice], a, pw, out=out, residual=residual, stream=stream, **kw)


# ----------------------------------------------------------------- table

@dataclass(frozen=True)
class DispatchEntry:
    n: int
    k: int
    m1: int
    m2: int

    def __post_init__(self):
        if not 1 <= self.m1 <= self.m2:
            raise ValueError(f"need 1 <= m1 <= m2, got m1={self.m1}, m2={self.m2}")


@dataclass
class DispatchTable:
    fingerprint: str
    version: str = TABLE_VERSION
    entries: dict = field(default_factory=dict)

    def add(self, entry: DispatchEntry):
        self.entries[(entry.n, entry.k)] = entry

    def lookup(self, n: int, k: int) -> DispatchEntry:
        try:
            return self.entries[(n, k)]
        except KeyError:
            raise UnknownShape(n, k) from None


def dispatch(m: int, n: int, k: int, table: DispatchTable) -> KernelChoice:
    """ImplA below M1, ImplB in [M1, M2), ImplC from M2 (dispatch.py:189-197);
    unknown (n, k) is an error, never a default."""
    e = table.lookup(n, k)
    return _FROM_CODE[_lib.load().fdpp_dispatch_choose(int(m), int(e.m1), int(e.m2))]


def dispatch_regret(table: DispatchTable, details: dict, tol: float = 1.10):
    """The reference's dispatch self-consistency criterion (test_acceptance.py:
    187-195): at every profiled point the dispatched kernel's median is within
    ``tol`` x the best of the three.  ``details`` maps "NxK" (or (n, k)) to the
    profile_shape rows.  Returns (worst ratio, [(n, k, m, picked, ratio) > tol])."""
    worst, bad = 1.0, []
    for key, rows in details.items():
        n, k = (int(x) for x in key.split("x")) if isinstance(key, str) else key
        for row in rows:
            picked = dispatch(row["m"], n, k, table).value
            best = min(row["ImplA"], row["ImplB"], row["ImplC"])
            ratio = row[picked] / best
            worst = max(worst, ratio)
            if ratio > tol:
                bad.append((n, k, row["m"], picked, round(ratio, 3)))
    return worst, bad


def default_fingerprint(workers: int = None) -> str:
    """B200 analogue of dispatch.py:200-203: device, SM count, lib ABI."""
    try:
        import torch
        name = torch.cuda.get_device_name().replace(" ", "_") if torch.cuda.is_available() else "nocuda"
    except Exception:
        name = "nocuda"
    sms = _lib.load().fdpp_sm_count()
    return f"{name}-sm{sms if sms > 0 else 'NA'}-fdpp{_lib.load().fdpp_version()}-cuda"


def save_table(table: DispatchTable, path) -> None:
    with open(path, "w") as f:
        f.write(f"{TABLE_MAGIC} {table.version} {table.fingerprint}\n")
        for (n, k) in sorted(table.entries):
            e = table.entries[(n, k)]
            f.write(f"{e.n} {e.k} {e.m1} {e.m2}\n")


def load_table(path, expected_fingerprint: str = None) -> DispatchTable:
    with open(path) as f:
        lines = f.read().splitlines()
    if not lines:
        raise ValueError(f"{path}:1: empty dispatch table file")
    head = lines[0].split(maxsplit=2)
    if len(head) != 3 or head[0] != TABLE_MAGIC:
        raise ValueError(f"{path}:1: bad header {lines[0]!r}")
    if head[1] != TABLE_VERSION:
        raise ValueError(f"{path}:1: unsupported version {head[1]!r} (want {TABLE_VERSION})")
    table = DispatchTable(fingerprint=head[2])
    for i, line in enumerate(lines[1:], start=2):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) != 4:
            raise ValueError(f"{path}:{i}: expected 'N K M1 M2', got {line!r}")
        try:
            n, k, m1, m2 = (int(v) for v in parts)
            table.add(DispatchEntry(n=n, k=k, m1=m1, m2=m2))
        except ValueError as exc:
            raise ValueError(f"{path}:{i}: {exc}") from None
    if expected_fingerprint is not None and table.fingerprint != expected_fingerprint:
        warnings.warn(
            f"dispatch table fingerprint {table.fingerprint!r} does not match "
            f"this environment ({expected_fingerprint!r}); timings may not transfer",
            stacklevel=2)
    return table


# ----------------------------------------------------------------- decision flow

def _dbl(xs):
    return (ctypes.c_double * len(xs))(*[float(x) for x in xs])


def _first_sustained(costs_new, costs_old, start=0):
    """dispatch.py:248-265 via fdpp_first_sustained; None when there is no win."""
    n = len(costs_new)
    i = _lib.load().fdpp_first_sustained(_dbl(costs_new), _dbl(costs_old), n, int(start))
    return None if i < 0 else i


def decide(m_sweep, med_a, med_b, med_c):
    """(m1, m2) from per-M medians (dispatch.py:326-338) via fdpp_profile_decide."""
    n = len(m_sweep)
    sweep = (ctypes.c_int32 * n)(*[int(m) for m in m_sweep])
    m1, m2 = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.load().fdpp_profile_decide(sweep, _dbl(med_a), _dbl(med_b), _dbl(med_c), n,
                                               ctypes.byref(m1), ctypes.byref(m2)), "profile")
    return m1.value, m2.value


def _time_impl(fn, reps, warmup, context, inner=1):
    """3 attempts, accept when MAD <= 0.2 * median (dispatch.py:268-275)."""
    for _ in range(3):
        samples = measure(fn, reps=reps, warmup=warmup, inner=inner)
        med, mad = median_mad(samples)
        if med == 0.0 or mad <= 0.2 * med:
            return med, mad
        warmup = 1
    raise TimingUnstable(f"timing noise above 20% of median for {context}")


def profile_shape(n: int, k: int, m_sweep=DEFAULT_M_SWEEP, reps: int = DEFAULT_REPS,
                  workers: int = None, warmup: int = DEFAULT_WARMUP, timers=None,
                  seed: int = 0, details: list = None, dtype=None) -> DispatchEntry:
    """Measure ImplA/B/C over an ascending M sweep on the device and locate the
    inflection points (dispatch.py:278-338).  ``timers`` substitutes analytic
    cost functions {name: f(m) -> seconds} (the fake-hardware hook used for
    bit-exact decision parity); ``details`` receives per-point medians."""
    m_sweep = list(m_sweep)
    if len(m_sweep) < 2 or any(b <= a for a, b in zip(m_sweep, m_sweep[1:])):
        raise ValueError("m_sweep must be ascending with at least 2 points")
    if reps < 3:
        raise ValueError("reps must be >= 3")
    names = [c.value for c in KernelChoice]
    medians = {name: [] for name in names}
    pws = None
    if timers is None:
        import torch
        _lib.require_cuda()
        dtype = dtype or torch.float16
        g = torch.Generator(device="cuda").manual_seed(seed)
        # enough weight copies that one timed batch streams >= 2x the 126 MB L2
        nbytes = n * k * 2
        nrot = max(1, min(16, -(-(256 << 20) // nbytes)))
        pws = []
        for _ in range(nrot):
            b = (torch.randn((k, n), generator=g, device="cuda") / np.sqrt(k)).to(dtype)
            pws.append(_g.pack_weight(b, dtype))
            del b
    for m in m_sweep:
        point = {"m": m}
        if timers is None:
            a = torch.randn((m, pws[0].ldw), generator=g, device="cuda").to(dtype)
            out = torch.empty((m, n), dtype=dtype, device="cuda")
            rot = [0]

            def mk(choice):
                def f():
                    run_device(choice, a, pws[rot[0] % len(pws)], out=out)
                    rot[0] += 1
                return f
            runs = {
                "ImplA": mk(KernelChoice.IMPL_A) if m <= GEMV_MAX_M else None,
                "ImplB": mk(KernelChoice.IMPL_B),
                "ImplC": mk(KernelChoice.IMPL_C),
            }
        for name in names:
            if timers is not None:
                med, mad = float(timers[name](m)), 0.0
            elif runs[name] is None:
                med, mad = float("inf"), 0.0
            else:
                med, mad = _time_impl(runs[name], reps, warmup, f"{name} at M={m} [N={n}, K={k}]",
                                      inner=len(pws))
            medians[name].append(med)
            point[name] = med
            point[f"{name}_mad"] = mad
        if details is not None:
            details.append(point)
    m1, m2 = decide(m_sweep, medians["ImplA"], medians["ImplB"], medians["ImplC"])
    return DispatchEntry(n=n, k=k, m1=m1, m2=m2)
