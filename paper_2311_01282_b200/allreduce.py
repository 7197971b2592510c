"""One-shot all-reduce fused into the row-parallel GEMM epilogue (SURVEY §8f
rank 2; the reference has no multi-GPU path).

Tensor-parallel O / down projections produce a partial [M, hidden] per rank
that must be summed across ranks.  Instead of GEMM -> ncclAllReduce, the
ImplB cluster epilogue pushes each CTA's fp32 output slice into every peer's
receive buffer with plain stores over peer memory (NVLink / NVSwitch),
publishes an epoch flag, waits for the peers' slices and writes the reduced
C (+ residual once, + the next RMSNorm's sums of squares) -- tile by tile,
overlapped with the other CTAs' MMAs (``fdpp_gemm_fuse.ar_*``,
include/fdpp.h).

``PeerAllReduce`` owns one rank's workspace (``fdpp_ar_alloc``: its own
cudaMalloc, so a CUDA IPC handle maps exactly it), exchanges IPC handles over
a torch.distributed group and maps the peers' workspaces.
``PeerAllReduce.local_group`` builds the same structure for several "ranks"
inside one process on one GPU (each rank's kernel on its own stream): the
single-GPU test of the exchange logic.
"""

from __future__ import annotations

import ctypes
from typing import List, Optional

from . import _lib

MAX_WORLD = _lib.AR_MAX_WORLD


def workspace_bytes(world: int, cap: int) -> int:
    n = ctypes.c_size_t()
    _lib.check(_lib.load().fdpp_ar_workspace_size(int(world), int(cap), ctypes.byref(n)), "ar_workspace_size")
    return n.value


class PeerAllReduce:
    """One rank's view: ``ptrs[r]`` = rank r's workspace mapped in this process."""

    def __init__(self, rank: int, world: int, cap: int, ptrs: List[int], owned: int, opened: List[int]):
        if not 2 <= world <= MAX_WORLD:
            raise ValueError(f"fused all-reduce needs 2..{MAX_WORLD} ranks, got {world}")
        self.rank, self.world, self.cap = rank, world, int(cap)
        self.ptrs = list(ptrs)
        self._owned = owned          # this process's own allocation (freed on close)
        self._opened = list(opened)  # IPC-mapped peer allocations (closed on close)

    # ---------------------------------------------------------------- creation
    @classmethod
    def create(cls, group, cap: int) -> "PeerAllReduce":
        """Collective over ``group`` (every rank calls it): allocate this rank's
        workspace for ``cap`` floats per receive slot (>= M * hidden), export
        its IPC handle, gather the peers' handles and map them."""
        import torch.distributed as dist
        lib = _lib.load()
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        ptr = ctypes.c_void_p()
        _lib.check(lib.fdpp_ar_alloc(workspace_bytes(world, cap), ctypes.byref(ptr)), "ar_alloc")
        h = ctypes.create_string_buffer(64)
        _lib.check(lib.fdpp_ipc_get_handle(ptr, h), "ipc_get_handle")
        handles: List[Optional[bytes]] = [None] * world
        dist.all_gather_object(handles, bytes(h.raw), group=group)
        ptrs, opened = [], []
        for r, hr in enumerate(handles):
            if r == rank:
                ptrs.append(ptr.value)
                continue
            p = ctypes.c_void_p()
            _lib.check(lib.fdpp_ipc_open(ctypes.create_string_buffer(hr, 64), ctypes.byref(p)), "ipc_open")
            ptrs.append(p.value)
            opened.append(p.value)
        return cls(rank, world, cap, ptrs, ptr.value, opened)

    @classmethod
    def local_group(cls, world: int, cap: int) -> List["PeerAllReduce"]:
        """``world`` ranks inside this process on the current GPU (no IPC)."""
        lib = _lib.load()
        ptrs = []
        for _ in range(world):
            p = ctypes.c_void_p()
            _lib.check(lib.fdpp_ar_alloc(workspace_bytes(world, cap), ctypes.byref(p)), "ar_alloc")
            ptrs.append(p.value)
        return [cls(r, world, cap, ptrs, ptrs[r], []) for r in range(world)]

    # ---------------------------------------------------------------- use
    def fill(self, fz) -> None:
        """Set the all-reduce fields of an fdpp_gemm_fuse."""
        fz.ar_rank, fz.ar_world, fz.ar_cap = self.rank, self.world, self.cap
        for r in range(MAX_WORLD):
            fz.ar_ws[r] = self.ptrs[r] if r < self.world else None

    def timed_out(self) -> bool:
        """True if a fused all-reduce on this rank gave up waiting for a peer."""
        t = ctypes.c_int32()
        _lib.check(_lib.load().fdpp_ar_check(ctypes.c_void_p(self.ptrs[self.rank]), ctypes.byref(t)), "ar_check")
        return bool(t.value)

    def close(self) -> None:
        lib = _lib.load()
        for p in self._opened:
            lib.fdpp_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        if self._owned:
            lib.fdpp_ar_free(ctypes.c_void_p(self._owned))
            self._owned = 0
