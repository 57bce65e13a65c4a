"""quantizer — SPEC `[MODULE] quantizer`: symmetric uniform quantization
(Eq. 1) with the scale layouts the kernels consume.

Host-side (offline) code.  Arithmetic is float32 with true IEEE division and
round-half-to-even, done with torch on any device, so weight codes are
bit-identical to the CPU reference contract (tests/test_host_api.py checks them against the
oracle).  The online activation quantizers live in the kernels (sq_quantize_f32,
sq_rmsnorm_quant, GEMM requant epilogues).

Weight formats (LEDGER G11):
* ``quantize_weight_w8``   PerChannel(axis=0) 8-bit          — W8A8 (int32 over all of K)
* ``quantize_weight_w4``   PerGroup(axis=1, 128) 4-bit float — W4A16 (SPEC literal)
* ``quantize_weight_w4a8`` the same SPEC PerGroup 4-bit weights; the A8 GEMM keeps one exact
  int32 accumulator per group and promotes it with the group's float scale (round 2; the
  round-1 progressive s_ch·sg scales measured worse SQNR, scripts/g11b_sqnr.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import LayoutError, ShapeError

__all__ = ["ScaleLayout", "QTensor", "compute_scale", "quantize", "dequantize", "fuse_scales",
           "quantize_weight_w8", "quantize_weight_w4", "quantize_weight_w4a8", "gptq_quantize_weight", "qrange"]


def qrange(bits: int):
    return -(1 << (bits - 1)), (1 << (bits - 1)) - 1


def _f32(x):
    return x.to(torch.float32) if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, np.float32))


def compute_scale(x_slice, bits: int, clip_percentile=None) -> float:
    """max|x| / (2^(b-1) - 1); 1.0 for an all-zero (or empty) slice."""
    if bits not in (4, 8):
        raise ValueError("bits must be 4 or 8")
    a = _f32(x_slice).abs().reshape(-1)
    if not bool(torch.isfinite(a).all()):
        raise ValueError("non-finite input")
    if a.numel() == 0:
        return np.float32(1.0)
    if clip_percentile is not None:
        m = np.float32(np.percentile(a.double().cpu().numpy(), clip_percentile))
    else:
        m = np.float32(a.max().item())
    if m == 0:
        return np.float32(1.0)
    return np.float32(m / np.float32(qrange(bits)[1]))


def _codes(x: torch.Tensor, s: torch.Tensor, bits: int) -> torch.Tensor:
    lo, hi = qrange(bits)
    return torch.round(x / s).clamp_(lo, hi).to(torch.int8)   # torch.round: half-to-even


@dataclass
class ScaleLayout:
    """SPEC.md:96-101.  kind ∈ {PerTensor, PerChannel, PerGroup, PerRow, Clustered,
    PerStateGroup}; ``scales`` f32.  Clustered carries ``cell_of`` (index -> cell)."""
    kind: str
    scales: object
    axis: int = -1
    group_size: int = 0
    bounds: tuple = ()
    cell_of: object = None

    def expand(self, shape) -> torch.Tensor:
        s = _f32(self.scales).reshape(-1)
        shape = tuple(shape)
        nd = len(shape)
        if bool((s <= 0).any()):
            raise LayoutError("scales must be > 0")
        if self.kind == "PerTensor":
            if s.numel() != 1:
                raise LayoutError("PerTensor needs one scale")
            return s.reshape(()).expand(shape)
        ax = 0 if self.kind == "PerRow" else self.axis % nd
        n = shape[ax]
        if self.kind == "PerGroup" and nd == 2 and ax == 1 and s.numel() == shape[0] * -(-n // self.group_size):
            g = torch.clamp(torch.arange(n) // self.group_size, max=s.numel() // shape[0] - 1)
            return s.reshape(shape[0], -1)[:, g]
        if self.kind in ("PerChannel", "PerRow"):
            idx = torch.arange(n)
        elif self.kind == "PerGroup":
            idx = torch.clamp(torch.arange(n) // self.group_size, max=s.numel() - 1)
        elif self.kind == "PerStateGroup":
            idx = torch.searchsorted(torch.as_tensor(self.bounds), torch.arange(n), right=True) - 1
        elif self.kind == "Clustered":
            idx = torch.as_tensor(np.asarray(self.cell_of), dtype=torch.long)
        else:
            raise LayoutError(f"unknown layout kind {self.kind}")
        if idx.numel() != n or int(idx.max()) >= s.numel():
            raise LayoutError("layout does not cover tensor")
        view = [1] * nd
        view[ax] = n
        return s[idx].reshape(view).expand(shape)


@dataclass
class QTensor:
    """integer payload (4-bit values kept unpacked as int8) + layout."""
    shape: tuple
    bits: int
    payload: torch.Tensor
    layout: ScaleLayout
    extra: dict = field(default_factory=dict)


def quantize(x, layout: ScaleLayout, bits: int) -> QTensor:
    """clamp(round_half_even(x / s))."""
    x = _f32(x)
    return QTensor(tuple(x.shape), bits, _codes(x, layout.expand(x.shape), bits), layout)


def dequantize(q: QTensor) -> torch.Tensor:
    """x̂ = q · s."""
    return q.payload.to(torch.float32) * q.layout.expand(q.shape)


def fuse_scales(s_x, s_w, s_y) -> np.float32:
    """s_fused = s_x / s_y; s_w rides in the weight scale."""
    if s_x <= 0 or s_w <= 0 or s_y <= 0:
        raise ValueError("scales must be > 0")
    return np.float32(np.float32(s_x) / np.float32(s_y))


def _group_absmax_scale(wg: torch.Tensor, bits: int) -> torch.Tensor:
    """compute_scale over the last axis of every group, vectorised (zero group -> 1.0)."""
    m = wg.abs().amax(dim=-1)
    s = m / np.float32(qrange(bits)[1])
    return torch.where(m == 0, torch.ones_like(s), s)


def quantize_weight_w8(w) -> QTensor:
    """PerChannel(axis=0) 8-bit weights (W8A8, LEDGER G11)."""
    w = _f32(w)
    if w.dim() != 2:
        raise ShapeError("weights are [out x in]")
    s = _group_absmax_scale(w, 8)
    codes = _codes(w, s[:, None], 8)
    return QTensor(tuple(w.shape), 8, codes, ScaleLayout("PerChannel", s, axis=0),
                   extra={"s_ch": s, "group": w.shape[1]})


def quantize_weight_w4(w, group: int = 128) -> QTensor:
    """PerGroup(axis=1, group) 4-bit weights with float scales (W4A16)."""
    w = _f32(w)
    n, k = w.shape
    if k % group:
        raise ShapeError("K must be a multiple of the group size")
    wg = w.reshape(n, k // group, group)
    s = _group_absmax_scale(wg, 4)
    codes = _codes(wg, s[:, :, None], 4).reshape(n, k)
    return QTensor((n, k), 4, codes, ScaleLayout("PerGroup", s.reshape(-1), axis=1, group_size=group),
                   extra={"s_group": s, "group": group})


def quantize_weight_w4a8(w, group: int = 128) -> QTensor:
    """W4A8 weights: SPEC PerGroup 4-bit with float group scales, the
    W4A16 format; only the activation precision differs (LEDGER G11)."""
    return quantize_weight_w4(w, group)


def gptq_quantize_weight(w, calib_inputs, bits: int = 4, group_size: int = 128, damp_ratio: float = 0.01,
                         device=None, block: int | None = None) -> QTensor:
    """SPEC.md:146-154 (GPTQ, Frantar et al.; PAPER.md Appendix "Implementation"): quantize the
    columns left to right, each group's scales recomputed per Eq. 1 over the group's CURRENT
    (error-compensated) weights, and every column's rounding error propagated to the columns on
    its right through the inverse Hessian H = 2·XᵀX + damp·I, damp = damp_ratio·mean(diag H).

    Runs on the GPU (``device``, default cuda when available): H and its inverse Cholesky factor
    in float64 (torch.linalg), the column sweep in float32 in blocks of ``block`` columns (default:
    the group size) whose accumulated errors update the remaining columns with one GEMM (the
    "lazy batch" form of the GPTQ paper).  A Hessian that stays singular after damping falls back
    to round-to-nearest (reported as a RuntimeWarning).  Returns the same QTensor
    layout as quantize_weight_w4 (bits 4) / PerGroup 8-bit (bits 8): codes int8 [out × in],
    scales [out × in/group]."""
    import warnings

    if bits not in (4, 8):
        raise ValueError("bits must be 4 or 8")
    dev = torch.device(device) if device is not None else (
        torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
    W = _f32(w).to(dev).clone()
    X = _f32(calib_inputs).to(dev)
    if W.dim() != 2 or X.dim() != 2 or X.shape[1] != W.shape[1] or X.shape[0] < 1:
        raise ShapeError("gptq: w [out x in], calib_inputs [samples x in] with samples >= 1")
    n_out, n_in = W.shape
    g = min(group_size, n_in)
    if n_in % g:
        raise ShapeError("gptq: group_size must divide in")
    qmax = float(qrange(bits)[1])
    lo, hi = qrange(bits)
    H = 2.0 * (X.double().T @ X.double())
    damp = damp_ratio * float(torch.diagonal(H).mean())
    H += damp * torch.eye(n_in, dtype=torch.float64, device=dev)
    try:
        Hinv = torch.cholesky_inverse(torch.linalg.cholesky(H))
        U = torch.linalg.cholesky(Hinv, upper=True).to(torch.float32)   # upper factor of H^-1
    except RuntimeError:   # torch.linalg raises on a non-positive-definite matrix
        warnings.warn("gptq: Hessian singular after damping; round-to-nearest for this layer", RuntimeWarning)
        return quantize_weight_w4(W, g) if bits == 4 else _rtn_per_group(W, g, bits)
    B = block or g
    codes = torch.empty((n_out, n_in), dtype=torch.int8, device=dev)
    scales = torch.empty((n_out, n_in // g), dtype=torch.float32, device=dev)
    for i0 in range(0, n_in, B):
        i1 = min(i0 + B, n_in)
        W1 = W[:, i0:i1].clone()
        E1 = torch.zeros_like(W1)
        U1 = U[i0:i1, i0:i1]
        for i in range(i1 - i0):
            col = i0 + i
            if col % g == 0:   # Eq. 1 over the group's current weights (its columns past this block
                # have received every earlier block's update; B is a multiple of g or g of B)
                grp = torch.cat([W1[:, i:], W[:, i1:col + g]], dim=1)[:, :g] if col + g > i1 else W1[:, i:i + g]
                m = grp.abs().amax(dim=1)
                s = torch.where(m == 0, torch.ones_like(m), m / np.float32(qmax))
                scales[:, col // g] = s
            s = scales[:, col // g]
            wc = W1[:, i]
            q = torch.round(wc / s).clamp_(lo, hi)
            codes[:, col] = q.to(torch.int8)
            err = (wc - q * s) / U1[i, i]
            if i + 1 < i1 - i0:
                W1[:, i + 1:] -= err[:, None] * U1[i, i + 1:][None, :]
            E1[:, i] = err
        if i1 < n_in:
            W[:, i1:] -= E1 @ U[i0:i1, i1:]
    return QTensor((n_out, n_in), bits, codes, ScaleLayout("PerGroup", scales.reshape(-1), axis=1, group_size=g),
                   extra={"s_group": scales, "group": g, "gptq": True})


def _rtn_per_group(w: torch.Tensor, group: int, bits: int) -> QTensor:
    n, k = w.shape
    wg = w.reshape(n, k // group, group)
    s = _group_absmax_scale(wg, bits)
    codes = _codes(wg, s[:, :, None], bits).reshape(n, k)
    return QTensor((n, k), bits, codes, ScaleLayout("PerGroup", s.reshape(-1), axis=1, group_size=group),
                   extra={"s_group": s, "group": group})
