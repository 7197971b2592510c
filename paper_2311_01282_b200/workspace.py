"""Per-device, per-stream zero-filled workspace pool for libfdpp.

The attention join counters and split-K tile counters live at the start of
the workspace; kernels leave them zeroed on exit, so a buffer is zero-filled
once at allocation and reused (and stays valid inside captured CUDA graphs).
"""

from __future__ import annotations

import threading

import torch

_lock = threading.Lock()
_pools: dict = {}


def get(nbytes: int, device=None, tag: str = "default") -> torch.Tensor:
    """A zero-initialised uint8 buffer of at least ``nbytes`` (grown, never shrunk).

    ``tag`` separates buffers that may be live at the same time on one stream
    (e.g. attention vs GEMM) or that a captured graph must own exclusively.
    """
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    # keyed by (device, tag), not by stream: a CUDA-graph capture must reuse the
    # buffer its warm-up allocated (an allocation inside capture would add a
    # zero-fill node to every replay).  Callers that run concurrently on
    # several streams pass distinct tags.
    key = (dev.index, tag)
    with _lock:
        buf = _pools.get(key)
        if buf is None or buf.numel() < max(nbytes, 1):
            size = max(int(nbytes * 1.25), 1 << 16)
            buf = torch.zeros(size, dtype=torch.uint8, device=dev)
            _pools[key] = buf
        return buf


def clear():
    with _lock:
        _pools.clear()
