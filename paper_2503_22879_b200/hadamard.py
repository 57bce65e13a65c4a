"""hadamard — SPEC `[MODULE] hadamard`, host side.

* ``fwht`` / ``fwht_blocked``: Sylvester butterflies in float32, stages h = 1, 2, 4, …
  (a+b, a-b) — the same stage order and f32 ops as the online transform inside the
  decode/prefill kernels (norm_had*_kernel, sq_gate_norm_had_quant), so host and device
  transforms are bit-identical.
* Non-power-of-two widths (LEDGER G9): block-diagonal I_q ⊗ H_b, b = largest power of two
  dividing n (5120 -> 5 x H_1024): orthogonal after 1/√b, exact for offline fusion,
  no Paley matrices.
* ``fuse_hadamard_out_proj`` / ``fuse_hadamard_in_proj``: offline weight
  rewrite in float64, normalised, so online transforms stay unnormalised.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import ShapeError
from .quantizer import _codes, _f32

__all__ = ["HadamardPlan", "fwht", "fwht_blocked", "fuse_hadamard_out_proj", "fuse_hadamard_in_proj",
           "hadamard_quantize", "hadamard_matrix", "block_size"]


def is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def block_size(n: int) -> int:
    return n & (-n)


@dataclass
class HadamardPlan:
    """SPEC.md:186-192."""
    n: int
    normalize: str = "none"        # "none" | "sqrt"
    fused_output_scale: float | None = None


def hadamard_matrix(n: int) -> torch.Tensor:
    if not is_pow2(n):
        raise ShapeError("n must be a power of two")
    h = torch.ones((1, 1), dtype=torch.int64)
    while h.shape[0] < n:
        h = torch.cat([torch.cat([h, h], 1), torch.cat([h, -h], 1)], 0)
    return h


def _butterflies(v: torch.Tensor) -> torch.Tensor:
    n = v.shape[-1]
    lead = v.shape[:-1]
    h = 1
    while h < n:
        r = v.reshape(*lead, n // (2 * h), 2, h)
        a, b = r[..., 0, :], r[..., 1, :]
        v = torch.stack([a + b, a - b], dim=-2).reshape(*lead, n)
        h *= 2
    return v


def fwht(v, plan: HadamardPlan) -> torch.Tensor:
    """Sylvester H_n along the last axis, then the plan's normalisation."""
    v = _f32(v)
    if v.shape[-1] != plan.n or not is_pow2(plan.n):
        raise ShapeError("fwht needs last dim == plan.n, a power of two")
    out = _butterflies(v)
    if plan.normalize == "sqrt":
        out = out * np.float32(1.0 / np.sqrt(plan.n))
    return out


def fwht_blocked(v, b: int | None = None) -> torch.Tensor:
    """Unnormalised I_q ⊗ H_b along the last axis (LEDGER G9; b = largest power of two dividing n
    by default, smaller for the shard-local transform of the head-shard recipe)."""
    v = _f32(v)
    n = v.shape[-1]
    b = block_size(n) if b is None else b
    return _butterflies(v.reshape(*v.shape[:-1], n // b, b)).reshape(v.shape)


def _blocked_matrix(n: int, b: int | None = None) -> np.ndarray:
    b = block_size(n) if b is None else b
    return np.kron(np.eye(n // b), hadamard_matrix(b).numpy().astype(np.float64)) / np.sqrt(b)


# The offline fusions use float64 numpy GEMMs (the reference's numeric stack, numpy>=1.24,
# pkg/pyproject.toml:10) so fused weights — hence weight codes — match the CPU contract bit
# for bit.
def fuse_hadamard_out_proj(w_out, n_in: int, n_out: int, block: int | None = None) -> torch.Tensor:
    """normalised H_out · W · H_inᵀ (n_out = 1 leaves the output side)."""
    w = np.asarray(w_out, np.float64)
    d_out, d_in = w.shape
    if n_in != d_in or n_out not in (1, d_out):
        raise ShapeError("fuse_hadamard_out_proj dims")
    r = w @ _blocked_matrix(d_in, block).T
    if n_out == d_out:
        r = _blocked_matrix(d_out) @ r
    return torch.from_numpy(r.astype(np.float32))


def fuse_hadamard_in_proj(w_in) -> torch.Tensor:
    """W · H̃ᵀ (normalised)."""
    w = np.asarray(w_in, np.float64)
    return torch.from_numpy((w @ _blocked_matrix(w.shape[1]).T).astype(np.float32))


def hadamard_quantize(y, plan: HadamardPlan, bits: int = 8, block: int | None = None) -> torch.Tensor:
    """quantize(H y, s_y) in one pass (unnormalised H, LEDGER G9 blocks)."""
    if plan.fused_output_scale is None:
        raise ValueError("missing fused scale")
    return _codes(fwht_blocked(y, block), torch.tensor(np.float32(plan.fused_output_scale)), bits)
