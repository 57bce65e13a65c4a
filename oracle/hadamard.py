"""Oracle: SPEC `[MODULE] hadamard`.

TEST INFRASTRUCTURE ONLY.

* ``fwht`` — Sylvester-ordered butterflies in float32, stages h = 1, 2, 4, …
  (a+b, a-b).  The GPU kernel runs the same stages with the same f32 ops, so
  its transform is bit-identical to this one.
* Non-power-of-two widths (LEDGER G9): the transform is block-diagonal
  ``I_q ⊗ H_b`` with b the largest power of two dividing n (5120 → 5×H_1024).
  It is orthogonal after 1/√b normalisation, needs no Paley matrices
   and keeps offline fusion exact.
* Online transform is unnormalised; 1/√b is folded into the fused weights
  (SPEC.md:238).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle.quantizer import quantize_codes


def is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def block_size(n: int) -> int:
    """Largest power of two dividing n (LEDGER G9)."""
    return n & (-n)


@dataclass
class HadamardPlan:
    n: int
    normalize: str = "none"          # "none" | "sqrt"
    fused_output_scale: float | None = None


def hadamard_matrix(n: int) -> np.ndarray:
    """Dense Sylvester H_n (integer ±1), n a power of two."""
    if not is_pow2(n):
        raise ValueError("n must be a power of two")
    h = np.ones((1, 1), dtype=np.int64)
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    return h


def _butterflies(v: np.ndarray) -> np.ndarray:
    v = np.array(v, dtype=np.float32, copy=True)
    n = v.shape[-1]
    lead = v.shape[:-1]
    h = 1
    while h < n:
        r = v.reshape(lead + (n // (2 * h), 2, h))
        a = r[..., 0, :]
        b = r[..., 1, :]
        v = np.stack([a + b, a - b], axis=-2).reshape(lead + (n,))
        h *= 2
    return v


def fwht(v, plan: HadamardPlan) -> np.ndarray:
    """SPEC.md:194-202 (power-of-two n only)."""
    v = np.asarray(v, np.float32)
    n = v.shape[-1]
    if n != plan.n or not is_pow2(n):
        from oracle.errors import ShapeError
        raise ShapeError("fwht needs last dim == plan.n, a power of two")
    out = _butterflies(v)
    if plan.normalize == "sqrt":
        out = (out * np.float32(1.0 / np.sqrt(n))).astype(np.float32)
    return out


def fwht_blocked(v, b: int | None = None) -> np.ndarray:
    """Unnormalised I_q ⊗ H_b along the last axis (LEDGER G9; b defaults to the largest power of
    two dividing n, a smaller power of two gives the shard-local transform)."""
    v = np.asarray(v, np.float32)
    n = v.shape[-1]
    b = block_size(n) if b is None else b
    r = v.reshape(v.shape[:-1] + (n // b, b))
    return _butterflies(r).reshape(v.shape)


def blocked_matrix(n: int, b: int | None = None) -> np.ndarray:
    b = block_size(n) if b is None else b
    return np.kron(np.eye(n // b, dtype=np.int64), hadamard_matrix(b))


def fuse_hadamard_out_proj(w_out, n_in: int, n_out: int, block: int | None = None) -> np.ndarray:
    """normalised H_out · W · H_inᵀ (block-diagonal for
    non-power-of-two widths; n_out = 1 leaves the output side unrotated)."""
    w = np.asarray(w_out, np.float64)
    d_out, d_in = w.shape
    if n_in != d_in or n_out not in (1, d_out):
        from oracle.errors import ShapeError
        raise ShapeError("fuse_hadamard_out_proj dims")
    bi = block_size(d_in) if block is None else block
    hi = blocked_matrix(d_in, bi) / np.sqrt(bi)
    r = w @ hi.T
    if n_out == d_out:
        ho = blocked_matrix(d_out) / np.sqrt(block_size(d_out))
        r = ho @ r
    return r.astype(np.float32)


def fuse_hadamard_in_proj(w_in) -> np.ndarray:
    """W · H̃ᵀ (normalised)."""
    w = np.asarray(w_in, np.float64)
    d_in = w.shape[1]
    h = blocked_matrix(d_in) / np.sqrt(block_size(d_in))
    return (w @ h.T).astype(np.float32)


def hadamard_quantize(y, plan: HadamardPlan, bits: int = 8, block: int | None = None) -> np.ndarray:
    """one-pass quantize(fwht(y), s_y) (unnormalised H)."""
    if plan.fused_output_scale is None:
        raise ValueError("missing fused scale")
    return quantize_codes(fwht_blocked(y, block), np.float32(plan.fused_output_scale), bits)
