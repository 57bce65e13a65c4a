"""Dense float32 tensors, a deterministic reference GEMM and seeded RNG streams.

Keeps the public API of the reference `pkg/src/ssmquant/tensor.py:12`
(``__all__``), with its defects fixed:
* D1 — ``make_rng`` built a 4-word Philox key and always raised; here the key is
  [seed, s0] and the counter [s1, s2, 0, 0] (LEDGER G1).
* D3 — ``ShapeError`` is the package-wide ``errors.ShapeError`` (still a ValueError).
* D4 — ``require_finite`` raises ``errors.ArchiveError`` (a ValueError).
``matmul`` is the reference float GEMM (tensor.py:33-54): host-side, used by the
offline calibration stages, never by the quantized GPU hot path.
"""
from __future__ import annotations

import numpy as np

from .errors import ArchiveError, ShapeError

__all__ = ["ShapeError", "as_f32", "require_finite", "matmul", "make_rng"]


def as_f32(x, shape=None) -> np.ndarray:
    """float32, C-contiguous view/copy of ``x`` (optionally reshaped)."""
    out = np.ascontiguousarray(x, dtype=np.float32)
    return out if shape is None else out.reshape(shape)


def require_finite(a: np.ndarray, name: str = "tensor") -> np.ndarray:
    """Reject NaN/Inf (archive invariant)."""
    if np.isfinite(a).all():
        return a
    raise ArchiveError(f"{name} contains non-finite values")


def matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Reference float GEMM: one float64 outer-product update per k, k ascending.

    Bit-identical to a scalar triple loop with the same order.
    """
    lhs, rhs = np.asarray(a), np.asarray(b)
    if lhs.ndim != 2 or rhs.ndim != 2:
        raise ShapeError(f"matmul needs 2-D operands, got {lhs.shape} and {rhs.shape}")
    if lhs.shape[1] != rhs.shape[0]:
        raise ShapeError(f"inner dimensions disagree: {lhs.shape} x {rhs.shape}")
    total = np.zeros((lhs.shape[0], rhs.shape[1]), dtype=np.float64)
    for col, row in zip(lhs.astype(np.float64).T, rhs.astype(np.float64)):
        total += np.multiply.outer(col, row)
    return total.astype(np.float32)


def make_rng(seed: int, *stream: int) -> np.random.Generator:
    """Counter-based deterministic generator (Philox), ≤3 substream keys."""
    if len(stream) > 3:
        raise ValueError("at most three substream keys are supported")
    s = [int(v) & 0xFFFFFFFFFFFFFFFF for v in stream] + [0, 0, 0]
    key = np.array([int(seed) & 0xFFFFFFFFFFFFFFFF, s[0]], dtype=np.uint64)
    counter = np.array([s[1], s[2], 0, 0], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key, counter=counter))
