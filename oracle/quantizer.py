"""Oracle: SPEC `[MODULE] quantizer` — symmetric uniform quant (Eq. 1).

TEST INFRASTRUCTURE ONLY.

All arithmetic is float32 with true IEEE division and round-half-to-even
(SPEC.md:122, 163): q = clamp(rint(x / s), -2^(b-1), 2^(b-1)-1).

Weight quantizers (LEDGER G11):
* ``quantize_weight_w8``       — PerChannel(axis=0) 8-bit, s[n] = max|w[n,:]|/127.
* ``quantize_weight_w4_group`` — PerGroup(axis=1, 128) 4-bit float scales
                                 (W4A16: SPEC literal).
* ``quantize_weight_w4a8``     — the same SPEC PerGroup 4-bit weights (float
                                 compute_scale per 128-group); the A8 GEMM keeps an
                                 exact int32 accumulator per group and promotes it
                                 with the group scale (LEDGER G11, round 2: replaces
                                 the round-1 progressive s_ch*sg scheme, which
                                 measured 0.14 dB worse toy-model SQNR and clamped
                                 small groups, scripts/g11b_sqnr.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def qrange(bits: int):
    return -(1 << (bits - 1)), (1 << (bits - 1)) - 1


def compute_scale(x_slice, bits: int, clip_percentile=None) -> np.float32:
    """max|x| / (2^(b-1)-1); 1.0 for an all-zero slice."""
    if bits not in (4, 8):
        raise ValueError("bits must be 4 or 8")
    a = np.abs(np.asarray(x_slice, dtype=np.float32))
    if not np.all(np.isfinite(a)):
        raise ValueError("non-finite input")
    if a.size == 0:
        return np.float32(1.0)
    m = np.float32(np.percentile(a, clip_percentile)) if clip_percentile is not None else np.float32(a.max())
    if m == 0:
        return np.float32(1.0)
    return np.float32(m / np.float32(qrange(bits)[1]))


def quantize_codes(x, s, bits: int) -> np.ndarray:
    """Element codes: clamp(rint(x/s)) in f32 (s broadcast to x)."""
    lo, hi = qrange(bits)
    q = np.rint(np.asarray(x, np.float32) / np.asarray(s, np.float32))
    return np.clip(q, lo, hi).astype(np.int8)


# --------------------------------------------------------------- layouts
@dataclass
class ScaleLayout:
    """SPEC.md:96-101.  kind in {PerTensor, PerChannel, PerGroup, PerRow,
    Clustered, PerStateGroup}; ``scales`` f32; ``axis``/``group_size``/
    ``bounds`` parametrise the kind.  For Clustered, ``cell_of`` maps each
    index along ``axis`` to a cell (expanded from a ClusterMap)."""
    kind: str
    scales: np.ndarray
    axis: int = -1
    group_size: int = 0
    bounds: tuple = ()
    cell_of: np.ndarray | None = None

    def expand(self, shape) -> np.ndarray:
        s = np.asarray(self.scales, np.float32)
        shape = tuple(shape)
        nd = len(shape)
        ax = self.axis % nd if nd else 0
        if np.any(s <= 0):
            from oracle.errors import LayoutError
            raise LayoutError("scales must be > 0")
        if self.kind == "PerTensor":
            return np.broadcast_to(s.reshape(()), shape)
        if self.kind == "PerGroup" and nd == 2 and ax == 1 and s.size == shape[0] * (-(-shape[1] // self.group_size)):
            # weight [out × in] with one scale per (row, group)
            g = np.minimum(np.arange(shape[1]) // self.group_size, s.size // shape[0] - 1)
            return s.reshape(shape[0], -1)[:, g]
        if self.kind == "PerRow":
            ax = 0
        if self.kind in ("PerChannel", "PerRow"):
            idx = np.arange(shape[ax])
        elif self.kind == "PerGroup":
            idx = np.arange(shape[ax]) // self.group_size
            if shape[ax] % self.group_size:
                idx = np.minimum(idx, s.size - 1)
        elif self.kind == "PerStateGroup":
            b = np.asarray(self.bounds)
            idx = np.searchsorted(b, np.arange(shape[ax]), side="right") - 1
        elif self.kind == "Clustered":
            idx = np.asarray(self.cell_of)
        else:
            raise ValueError(f"unknown layout kind {self.kind}")
        if idx.max(initial=-1) >= s.size or len(idx) != shape[ax]:
            from oracle.errors import LayoutError
            raise LayoutError("layout does not cover tensor")
        v = s[idx]
        bshape = [1] * nd
        bshape[ax] = shape[ax]
        return np.broadcast_to(v.reshape(bshape), shape)


@dataclass
class QTensor:
    """integer payload + layout."""
    shape: tuple
    bits: int
    payload: np.ndarray          # int8 codes (4-bit values stored unpacked as int8)
    layout: ScaleLayout
    extra: dict = field(default_factory=dict)


def quantize(x, layout: ScaleLayout, bits: int) -> QTensor:
    """SPEC.md:119-127."""
    x = np.asarray(x, np.float32)
    s = layout.expand(x.shape)
    return QTensor(x.shape, bits, quantize_codes(x, s, bits), layout)


def dequantize(q: QTensor) -> np.ndarray:
    """x = q * s."""
    s = q.layout.expand(q.shape)
    return (q.payload.astype(np.float32) * s).astype(np.float32)


def fuse_scales(s_x, s_w, s_y) -> np.float32:
    """s_fused = s_x / s_y (s_w kept for the signature)."""
    if s_x <= 0 or s_w <= 0 or s_y <= 0:
        raise ValueError("scales must be > 0")
    return np.float32(np.float32(s_x) / np.float32(s_y))


# ------------------------------------------------------- weight quantizers
def quantize_weight_w8(w) -> QTensor:
    """PerChannel(axis=0) 8-bit weights (G11: W8A8 per-output-channel)."""
    w = np.asarray(w, np.float32)
    s = np.array([compute_scale(w[n], 8) for n in range(w.shape[0])], np.float32)
    lay = ScaleLayout("PerChannel", s, axis=0)
    return QTensor(w.shape, 8, quantize_codes(w, s[:, None], 8), lay,
                   extra={"s_ch": s, "group": w.shape[1]})


def quantize_weight_w4_group(w, group: int = 128) -> QTensor:
    """PerGroup(axis=1, group) 4-bit with float scales (W4A16, SPEC literal)."""
    w = np.asarray(w, np.float32)
    n, k = w.shape
    if k % group:
        raise ValueError("K must be a multiple of group")
    g = k // group
    wg = w.reshape(n, g, group)
    s = np.empty((n, g), np.float32)
    for i in range(n):
        for j in range(g):
            s[i, j] = compute_scale(wg[i, j], 4)
    lay = ScaleLayout("PerGroup", s.reshape(-1), axis=1, group_size=group)
    codes = quantize_codes(wg, s[:, :, None], 4).reshape(n, k)
    return QTensor(w.shape, 4, codes, lay, extra={"s_group": s, "group": group})


def quantize_weight_w4a8(w, group: int = 128) -> QTensor:
    """W4A8 weights: SPEC PerGroup 4-bit with float scales, the same
    format as W4A16; only the activation precision differs (LEDGER G11)."""
    return quantize_weight_w4_group(w, group)
