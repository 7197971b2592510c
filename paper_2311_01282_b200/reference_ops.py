"""Float64 reference modes on the device (the reference's oracle-side API:
``gemm_oracle`` matrix.py:90-104 and ``attention_reference`` attention.py:77-86,
reached through ``batch_decode_attention(..., "reference")``).

These are the *reference* modes of the drop-in API, not the hot path: they
run in float64 on the GPU (FP64 pipe) so a caller of the reference's
"reference" mode gets the same all-f64 semantics without a CPU detour.
"""

from __future__ import annotations

import numpy as np


def attention_f64(Q, K, V, scale: float):
    q, k, v = Q.double(), K.double(), V.double()
    s = scale * (q @ k.T)
    e = (s - s.max(dim=1, keepdim=True).values).exp()
    return ((e / e.sum(dim=1, keepdim=True)) @ v).float()


def gemm_oracle(a, b):
    """f64 accumulation, rounded once to f32 (matrix.py:90-104)."""
    import torch
    from . import _lib
    was_numpy = not isinstance(a, torch.Tensor)
    _lib.require_cuda()
    A = torch.as_tensor(np.asarray(a, np.float32) if was_numpy else a).cuda().double()
    B = torch.as_tensor(np.asarray(b, np.float32) if was_numpy else b).cuda().double()
    if A.shape[1] != B.shape[0]:
        from .matrix import ShapeError
        raise ShapeError(f"inner dims disagree: {tuple(A.shape)} x {tuple(B.shape)}")
    c = (A @ B).float()
    return c.cpu().numpy() if was_numpy else c
