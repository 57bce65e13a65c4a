"""calibrate — SPEC `[MODULE] calibrate`, host side (offline).

Produces the runtime tables the kernels read: the sort-and-cluster ClusterMap for x
(PAPER.md:207-219), per-state-group B/C scales and the cached-state scales over the
ClusterMap cells (LEDGER G7).

Ledgered choices, shared with the test oracle so cluster indices are
bit-exact (tests/test_host_api.py):
* head feature = the head's descending-sorted channel-max vector;
* k-means++ init from ``make_rng(seed, 0x6B6D)``, <= 100 Lloyd iterations, ties -> lowest
  centre, an empty cluster keeps its centre; distances in float64;
* clusters ordered by their smallest original head index, heads inside a cluster by index;
* channel groups: 1-D k-means over the pooled sorted maxima (non-increasing, so every
  cluster is a contiguous run of sorted positions); fewer distinct points than clusters ->
  equal-size contiguous groups.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import CalibrationError, ShapeError
from .quantizer import compute_scale
from .tensor import make_rng

__all__ = ["CalibStats", "ClusterMap", "StateGroupScales", "stats_of", "kmeans", "sort_and_cluster",
           "build_state_group_scales", "calibrate_site_scale", "collect_stats"]

KMEANS_STREAM = 0x6B6D


@dataclass
class CalibStats:
    """per-channel running max of |activation| (+ optional sorted values
    for percentile clipping).  ``merge`` is order-independent (max / sorted union)."""
    channel_max: np.ndarray
    sample_count: int = 0
    values: np.ndarray | None = None

    def merge(self, other: "CalibStats") -> "CalibStats":
        v = None
        if self.values is not None and other.values is not None:
            v = np.sort(np.concatenate([self.values, other.values]))
        return CalibStats(np.maximum(self.channel_max, other.channel_max), self.sample_count + other.sample_count, v)


def stats_of(act, channel_shape, keep_values=False) -> CalibStats:
    a = torch.as_tensor(act).detach().to(torch.float32).abs().reshape((-1,) + tuple(channel_shape))
    cm = a.amax(dim=0).cpu().numpy() if a.shape[0] else np.zeros(channel_shape, np.float32)
    vals = np.sort(a.reshape(-1).cpu().numpy()) if keep_values else None
    return CalibStats(cm.astype(np.float32), a.shape[0], vals)


@dataclass
class ClusterMap:
    """SPEC.md:371-377."""
    head_perm: np.ndarray            # [nh] new position -> old head
    channel_perm: np.ndarray         # [nh, P] per OLD head: sorted position -> old channel
    head_group_bounds: np.ndarray    # [m+1]
    channel_group_bounds: np.ndarray  # [m, n+1]
    scales: np.ndarray               # [m, n]

    @property
    def m(self):
        return len(self.head_group_bounds) - 1

    @property
    def n(self):
        return self.channel_group_bounds.shape[1] - 1

    def cell_of_new(self) -> np.ndarray:
        """Cell (i*n + j) of every channel of the REORDERED layout [nh*P]."""
        nh, P = self.channel_perm.shape
        cells = np.empty(nh * P, np.int32)
        for i in range(self.m):
            lo_h, hi_h = self.head_group_bounds[i], self.head_group_bounds[i + 1]
            for j in range(self.n):
                lo, hi = self.channel_group_bounds[i, j], self.channel_group_bounds[i, j + 1]
                for hp in range(lo_h, hi_h):
                    cells[hp * P + lo:hp * P + hi] = i * self.n + j
        return cells


@dataclass
class StateGroupScales:
    """SPEC.md:378-381."""
    boundaries: np.ndarray
    scales_B: np.ndarray
    scales_C: np.ndarray
    scales_state: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


def kmeans(X, k: int, seed: int = 0, iters: int = 100) -> np.ndarray:
    """Lloyd k-means with k-means++ init (float64), labels [n]."""
    X = np.asarray(X, np.float64)
    n = X.shape[0]
    rng = make_rng(seed, KMEANS_STREAM)
    first = int(rng.integers(n))
    centers = [X[first].copy()]
    d2 = ((X - centers[0]) ** 2).sum(axis=1)
    for _ in range(1, k):
        tot = d2.sum()
        if tot <= 0:
            centers.append(X[first].copy())
        else:
            r = rng.random() * tot
            idx = int(np.searchsorted(np.cumsum(d2), r, side="right"))
            centers.append(X[min(idx, n - 1)].copy())
        d2 = np.minimum(d2, ((X - centers[-1]) ** 2).sum(axis=1))
    C = np.array(centers)
    labels = np.full(n, -1)
    for _ in range(iters):
        dist = ((X[:, None, :] - C[None, :, :]) ** 2).sum(axis=2)
        new = dist.argmin(axis=1)                 # first minimum -> lowest centre on ties
        if np.array_equal(new, labels):
            break
        labels = new
        for j in range(k):
            mem = labels == j
            if mem.any():
                C[j] = X[mem].mean(axis=0)
    return labels


def _equal_groups(count: int, k: int) -> np.ndarray:
    return (np.arange(count) * k) // count


def sort_and_cluster(stats_x: CalibStats, n_heads: int, head_dim: int, m: int = 4, n: int = 4, seed: int = 0,
                     bits: int = 8) -> ClusterMap:
    """SPEC.md:393-401 (defaults m = n = 4; scaled to the toy dims)."""
    mx = np.asarray(stats_x.channel_max, np.float32).reshape(n_heads, head_dim)
    m, n = min(m, n_heads), min(n, head_dim)
    cperm = np.argsort(-mx, axis=1, kind="stable").astype(np.int64)
    F = np.take_along_axis(mx, cperm, axis=1)
    labels = _equal_groups(n_heads, m) if len(np.unique(F, axis=0)) < m else kmeans(F, m, seed)
    order = sorted(set(labels.tolist()), key=lambda l: int(np.flatnonzero(labels == l)[0]))
    head_perm = np.concatenate([np.flatnonzero(labels == l) for l in order]).astype(np.int64)
    hb = np.concatenate([[0], np.cumsum([int((labels == l).sum()) for l in order])]).astype(np.int64)
    cb = np.zeros((len(order), n + 1), np.int64)
    scales = np.zeros((len(order), n), np.float32)
    for i in range(len(order)):
        heads = head_perm[hb[i]:hb[i + 1]]
        v = F[heads].max(axis=0)
        lab = _equal_groups(head_dim, n) if len(np.unique(v)) < n else kmeans(v[:, None], n, seed)
        cuts = list(np.flatnonzero(np.diff(lab)) + 1)
        if len(cuts) != n - 1:
            lab = _equal_groups(head_dim, n)
            cuts = list(np.flatnonzero(np.diff(lab)) + 1)
        cb[i] = [0] + cuts + [head_dim]
        for j in range(n):
            scales[i, j] = compute_scale(F[heads][:, cb[i, j]:cb[i, j + 1]], bits)
    return ClusterMap(head_perm, cperm, hb, cb, scales)


def build_state_group_scales(stats_B: CalibStats, stats_C: CalibStats, n_state_groups: int, d_state: int,
                             stats_h: CalibStats | None = None, cmap: ClusterMap | None = None,
                             bits: int = 8) -> StateGroupScales:
    """SPEC.md:402-410; with ``stats_h`` and ``cmap`` also the cached-state scales over the
    ClusterMap cells in the reordered layout (LEDGER G7)."""
    mb = np.asarray(stats_B.channel_max, np.float32).reshape(n_state_groups, d_state)
    mc = np.asarray(stats_C.channel_max, np.float32).reshape(n_state_groups, d_state)
    sB = np.array([compute_scale(mb[g], bits) for g in range(n_state_groups)], np.float32)
    sC = np.array([compute_scale(mc[g], bits) for g in range(n_state_groups)], np.float32)
    ss = None
    if stats_h is not None and cmap is not None:
        nh, P = cmap.channel_perm.shape
        hm = np.asarray(stats_h.channel_max, np.float32).reshape(nh, P)
        hp = np.asarray(cmap.head_perm)
        hm_new = np.take_along_axis(hm[hp], np.asarray(cmap.channel_perm)[hp], axis=1)
        cells = cmap.cell_of_new().reshape(nh, P)
        ss = np.ones((cmap.m, cmap.n), np.float32)
        for c in range(cmap.m * cmap.n):
            ss.reshape(-1)[c] = compute_scale(hm_new[cells == c], bits)
    return StateGroupScales(np.arange(n_state_groups + 1) * d_state, sB, sC, ss)


def calibrate_site_scale(stats: CalibStats, bits: int = 8, clip_percentile=None) -> np.float32:
    """SPEC.md:411-419."""
    if stats.sample_count == 0 and not np.any(stats.channel_max):
        return np.float32(1.0)
    if clip_percentile is not None and stats.values is not None and stats.values.size:
        return compute_scale(stats.values, bits, clip_percentile)
    return compute_scale(stats.channel_max, bits)


SITES = ("u", "z", "x_in", "B_in", "C_in", "dt", "x", "B", "C", "h", "dt_low", "y", "r", "y_had", "head_in")


ROW_SITES = ("u", "x", "dt_low", "r")   # projection inputs: in_proj, x_proj, dt_proj, out_proj


def collect_stats(model, tokens, sites=None, device="cuda", keep_rows: int = 0):
    """per layer, per calibration site, channel maxima over all samples.
    Runs the float model (``float_path.float_forward``) on ``device``; returns one dict of
    CalibStats per block plus the head input site at index -1.  ``sites``
    restricts the taps kept (names in ``SITES``); None keeps every site.  ``keep_rows`` > 0 also
    keeps the first ``keep_rows`` activation rows of every projection input (``ROW_SITES``, on
    ``device``) under ``stats[l]["_rows"]``: the calibration inputs of GPTQ."""
    if sites is not None:
        unknown = set(sites) - set(SITES)
        if unknown:
            raise CalibrationError(f"unknown calibration sites {sorted(unknown)}")
    from .float_path import float_forward
    tokens = np.asarray(tokens)
    if tokens.ndim != 2 or tokens.shape[0] == 0:
        raise CalibrationError("calibration set must be [samples x T] with >= 1 sample")
    L = len(model.blocks)
    stats = [dict() for _ in range(L + 1)]
    for s in range(tokens.shape[0]):
        taps = []
        float_forward(model, tokens[s], taps, device=device)
        for l in range(L + 1):
            if keep_rows > 0 and l < L:
                rows = stats[l].setdefault("_rows", {})
                for k in ROW_SITES:
                    if k in taps[l]:
                        have = rows.get(k)
                        need = keep_rows - (0 if have is None else have.shape[0])
                        if need > 0:
                            v = taps[l][k][:need].detach()
                            rows[k] = v if have is None else torch.cat([have, v])
            for k, v in taps[l].items():
                if sites is not None and k not in sites:
                    continue
                ch = tuple(v.shape) if k == "h" else tuple(v.shape[1:])
                st = stats_of(v[None] if k == "h" else v, ch)
                stats[l][k] = st if k not in stats[l] else stats[l][k].merge(st)
    if sites is None and any(not [k for k in s if k != "_rows"] for s in stats):
        raise ShapeError("calibration produced no statistics")
    return stats
