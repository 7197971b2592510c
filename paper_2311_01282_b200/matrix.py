"""Matrix invariants and shapes (reference: flatdecode/matrix.py).

Host-side helpers kept API-compatible with the reference: ``ShapeError``
(matrix.py:16), ``GemmShape`` (:20), ``validate_shape`` (:26), ``as_matrix``
(:32) and ``pad_rows`` (:53).  ``gemm_oracle`` (:90) is provided on the device
in float64 (see ``reference_ops``); binary matrix files are out of scope.
"""

from typing import NamedTuple

import numpy as np


class ShapeError(ValueError):
    pass


class GemmShape(NamedTuple):
    m: int
    n: int
    k: int


def validate_shape(shape: GemmShape) -> GemmShape:
    if shape.m < 1 or shape.n < 1 or shape.k < 1:
        raise ShapeError(f"GEMM dims must be >= 1, got {shape}")
    return shape


def as_matrix(data, rows: int = None, cols: int = None, checked: bool = True) -> np.ndarray:
    a = np.ascontiguousarray(data, dtype=np.float32)
    if rows is not None or cols is not None:
        if rows is None or cols is None:
            raise ShapeError("rows and cols must be given together")
        a = a.reshape(rows, cols)
    if a.ndim != 2:
        raise ShapeError(f"matrix must be 2-D, got ndim={a.ndim}")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise ShapeError(f"matrix dims must be >= 1, got {a.shape}")
    if checked and not np.isfinite(a).all():
        bad = np.argwhere(~np.isfinite(a))[0]
        raise ValueError(f"non-finite element at ({bad[0]}, {bad[1]})")
    return a


def pad_rows(a, multiple: int):
    """Zero-pad rows to a multiple; aligned input is returned as-is (works on
    numpy arrays and torch tensors)."""
    if multiple < 1:
        raise ValueError("padding multiple must be >= 1")
    rows = a.shape[0]
    padded = ((rows + multiple - 1) // multiple) * multiple
    if padded == rows:
        return a
    if isinstance(a, np.ndarray):
        out = np.zeros((padded, a.shape[1]), dtype=np.float32)
    else:
        import torch
        out = torch.zeros((padded, a.shape[1]), dtype=a.dtype, device=a.device)
    out[:rows] = a
    return out
