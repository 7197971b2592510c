"""Flat GEMM (reference: flatdecode/flatgemm.py).

Host-side model kept verbatim in behaviour: ``TileConfig`` (flatgemm.py:23-32),
``CostEstimate`` / ``arithmetic_intensity`` (Eq. (5), :35-69), ``select_tile``
(:72-102) and ``double_buffer_pipeline`` (:107-126).

``flat_gemm`` (:215-242) runs the B200 ImplB kernel: swap-AB tcgen05 with the
weight tile on the 128-row MMA M axis and the M <= 64 tokens on the MMA N axis
(TMA zero-fills the padded token rows: the paper's "pad to 8" with no padded
copy).  TileConfig maps onto the device tile as follows: ``double_buffer`` ->
a 2-stage TMA ring (else 1 stage, the single-buffer schedule); ``m_pad`` -> the
token tile (rounded up to 16/32/64, the legal MMA N sizes); ``b_n`` / ``b_k``
are CPU cache-blocking parameters with no device meaning (the device tile is
128 x 64, one SWIZZLE_128B atom wide).  ``flat_gemm_b200`` exposes the
device knobs directly (token tile, persistent grid, ring depth).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import gemm as _g
from .matrix import GemmShape, ShapeError, validate_shape

MICROKERNEL_ROWS = 8
MICROKERNEL_WIDTH = 8
DEFAULT_B_K = 32
B200_SMS = 148


@dataclass(frozen=True)
class TileConfig:
    b_n: int
    b_k: int
    m_pad: int = MICROKERNEL_ROWS
    double_buffer: bool = False

    def __post_init__(self):
        if self.b_n < 1 or self.b_k < 1 or self.m_pad < 1:
            raise ValueError(f"tile sizes must be >= 1, got {self}")


@dataclass(frozen=True)
class CostEstimate:
    """Work and traffic of one tiled flat GEMM (``bytes`` counts elements,
    as in the reference, flatgemm.py:35-46)."""

    flops: int
    bytes: float
    intensity: float
    parallelism: float


def arithmetic_intensity(shape: GemmShape, b_n: int, b_k: int) -> CostEstimate:
    """Eq. (5) cost model (flatgemm.py:49-69)."""
    validate_shape(shape)
    m, n, k = shape
    if not (1 <= b_n <= n and 1 <= b_k <= k):
        raise ValueError(f"invalid tile ({b_n}, {b_k}) for shape {shape}")
    flops = 2 * m * n * k
    n_tiles = (n * k) / (b_n * b_k)
    traffic = (m * b_k + b_n * b_k) * n_tiles + m * n
    return CostEstimate(flops=flops, bytes=traffic, intensity=flops / traffic, parallelism=n / b_n)


def _width_candidates(n: int):
    cands = [w for w in (1, 2, 4) if w <= n]
    cands += list(range(MICROKERNEL_WIDTH, n + 1, MICROKERNEL_WIDTH))
    return cands


def select_tile(shape: GemmShape, workers: int, parallel_target: int = None) -> TileConfig:
    """Tile heuristic (flatgemm.py:78-102); ``workers`` = 148 SMs on B200."""
    validate_shape(shape)
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if parallel_target is None:
        parallel_target = 4 * workers
    n, k = shape.n, shape.k
    b_k = min(DEFAULT_B_K, k)
    cands = _width_candidates(n)
    if n <= parallel_target * MICROKERNEL_WIDTH:
        feasible = [w for w in cands if n / w >= workers] or cands
        b_n = min(feasible, key=lambda w: (abs(n / w - parallel_target), w))
        return TileConfig(b_n=b_n, b_k=b_k, double_buffer=False)
    feasible = [w for w in cands if n / w >= workers]
    return TileConfig(b_n=max(feasible), b_k=b_k, double_buffer=True)


def double_buffer_pipeline(n_k_tiles: int):
    """Double-buffer event schedule (flatgemm.py:107-126)."""
    return ring_pipeline(n_k_tiles, 2)


def ring_pipeline(n_k_tiles: int, stages: int):
    """Event schedule of the S-stage TMA/mbarrier ring the B200 kernel runs:
    the producer keeps S tiles in flight and refills slot t % S with tile
    t + S only after compute(t) has released it (the mbarrier 'empty' wait).
    stages == 2 is exactly the reference's double buffer."""
    if n_k_tiles < 1:
        raise ValueError("need at least one K tile")
    if stages < 1:
        raise ValueError("need at least one stage")
    events = [("fill", t, t % stages) for t in range(min(stages, n_k_tiles))]
    for t in range(n_k_tiles):
        events.append(("compute", t, t % stages))
        if t + stages < n_k_tiles:
            events.append(("fill", t + stages, (t + stages) % stages))
    return events


def _token_tile(m_pad: int, M: int) -> int:
    want = max(m_pad, M)
    return 16 if want <= 16 else 32 if want <= 32 else 64


def flat_gemm(a, b, cfg: TileConfig, record_events=None):
    """ImplB on the device; same contract as flatgemm.py:215-242 (M padding is
    transparent, double buffering never changes bits)."""
    K = b.K if isinstance(b, _g.PackedWeight) else b.shape[0]
    if a.shape[1] != K:
        raise ShapeError(f"inner dims disagree: {tuple(a.shape)} x {tuple(getattr(b, 'shape', ()))}")
    M = a.shape[0]
    stages = 2 if cfg.double_buffer else 1
    bx = _token_tile(cfg.m_pad, min(M, 64))
    if record_events is not None:
        n_tiles = -(-(b.N if isinstance(b, _g.PackedWeight) else b.shape[1]) // 128)
        k_tiles = -(-K // 64)
        for nt in range(n_tiles):
            for op, kt, buf in ring_pipeline(k_tiles, stages):
                record_events.append((op, nt, kt, buf))
    return _g.reference_call(_g.IMPL_B, a, b, block_x=bx, stages=stages)


def flat_gemm_b200(a, b, *, block_x: int = 0, ctas: int = 0, stages: int = 0, out=None,
                   residual=None, stream=None):
    """ImplB with the device knobs exposed (0 = auto): token tile, persistent
    grid size (stream-K CTAs), ring depth."""
    return _g.reference_call(_g.IMPL_B, a, b, block_x=block_x, ctas=ctas, stages=stages,
                             out=out, residual=residual, stream=stream)
