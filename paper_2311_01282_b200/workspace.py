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


def get(nbytes: int, device=None, tag: str = "default", stream=None) -> torch.Tensor:
    """A zero-initialised uint8 buffer of at least ``nbytes`` (grown, never shrunk).

    ``tag`` separates buffers that may be live at the same time on one stream
    (e.g. attention vs GEMM) or that a captured graph must own exclusively.
    ``stream`` is the stream the caller launches on (default: the current
    stream): a new buffer is zero-filled on it, and the buffer is recorded on
    every stream it is handed to, so growing it never frees memory a kernel
    on another stream may still be using.
    """
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    # keyed by (device, tag), not by stream: a CUDA-graph capture must reuse the
    # buffer its warm-up allocated (an allocation inside capture would add a
    # zero-fill node to every replay).  Callers that run concurrently on
    # several streams pass distinct tags.
    key = (dev.index, tag)
    with _lock:
        ent = _pools.get(key)
        if ent is None or ent[0].numel() < max(nbytes, 1):
            size = max(int(nbytes * 1.25), 1 << 16)
            with torch.cuda.stream(s):   # zero-filled in the launch stream's order
                buf = torch.zeros(size, dtype=torch.uint8, device=dev)
            ent = (buf, {s.cuda_stream})
            _pools[key] = ent          # the old buffer was recorded on its streams
        buf, used = ent
        # (not during graph capture: the captured graph keeps its buffer alive)
        if s.cuda_stream not in used and not torch.cuda.is_current_stream_capturing():
            buf.record_stream(s)
            used.add(s.cuda_stream)
        return buf


def clear():
    with _lock:
        _pools.clear()
