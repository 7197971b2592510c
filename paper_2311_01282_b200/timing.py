"""Device-side timing for the profiler and bench (reference: flatdecode/timing.py).

``median_mad`` keeps the reference's definition (timing.py:8-13).
``measure`` replaces the wall clock (timing.py:16-25) with CUDA events on the
launching stream, synchronised on both sides, and flushes L2 before each
timed rep so a kernel never reports cache bandwidth as HBM bandwidth.
"""

from __future__ import annotations

import numpy as np
import torch

_FLUSH = {}


def median_mad(samples):
    s = np.asarray(samples, dtype=np.float64)
    med = float(np.median(s))
    mad = float(np.median(np.abs(s - med)))
    return med, mad


def l2_flush(device=None, nbytes: int = 256 << 20):
    """READ a buffer twice the 126 MB L2 so the next kernel starts cold.

    A read (not a memset) leaves L2 holding clean lines, as it would after
    the previous layer's weight stream; a write-flush would make the timed
    kernel pay for writing back ~126 MB of dirty lines."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    ent = _FLUSH.get(dev.index)
    if ent is None or ent[0].numel() * 4 < nbytes:
        ent = (torch.ones(nbytes // 4, dtype=torch.float32, device=dev),
               torch.empty((), dtype=torch.float32, device=dev))
        _FLUSH[dev.index] = ent
    torch.sum(ent[0], dim=0, out=ent[1])


SPIN_CYCLES = 400_000   # ~0.2-0.3 ms at B200 clocks: longer than any host launch path


def measure(fn, reps: int, warmup: int = 2, flush_l2: bool = True, inner: int = 1):
    """Seconds per call of fn(), one CUDA-event pair per rep, after warmup.

    Before each rep the stream is parked on a spin kernel, so fn()'s launches
    are already queued when the start event fires: the host launch latency
    (Python -> ctypes -> libfdpp) never leaks into the device-timed window.
    ``inner`` > 1 times that many back-to-back calls per rep and divides (the
    event clock ticks in ~2 us steps on this part; a longer window resolves
    sub-tick differences).  Callers that pass inner > 1 must rotate operands
    so consecutive calls do not hit in L2."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    out = []
    stream = torch.cuda.current_stream()
    for _ in range(reps):
        if flush_l2:
            l2_flush()
        torch.cuda._sleep(SPIN_CYCLES)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(inner):
            fn()
        e1.record(stream)
        e1.synchronize()
        out.append(e0.elapsed_time(e1) * 1e-3 / inner)
    return out
