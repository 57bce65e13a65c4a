"""Oracle: SPEC `[MODULE] calibrate`.

TEST INFRASTRUCTURE ONLY.

Ledgered choices:
* head feature = the head's descending-sorted channel-max vector;
* k-means: k-means++ init from ``make_rng(seed, 0x6B6D)``, ≤100 Lloyd
  iterations, ties → lowest centre index, empty cluster keeps its centre;
* clusters ordered by their smallest original head index; heads inside a
  cluster by original index;
* channel groups: 1-D k-means (k=n) over v_p = max_{h∈group} sorted_max[h,p],
  which is non-increasing in p, so every cluster is a contiguous run of
  sorted positions;
* fallback: fewer distinct points than clusters → equal-size contiguous groups.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from oracle.quantizer import compute_scale
from oracle.tensor_core import make_rng

KMEANS_STREAM = 0x6B6D


@dataclass
class CalibStats:
    """per-channel running max of |·| (channel axis = trailing dims)."""
    channel_max: np.ndarray
    sample_count: int = 0
    values: np.ndarray | None = None      # optional percentile sketch

    def merge(self, other: "CalibStats") -> "CalibStats":
        v = None
        if self.values is not None and other.values is not None:
            v = np.sort(np.concatenate([self.values, other.values]))
        return CalibStats(np.maximum(self.channel_max, other.channel_max),
                          self.sample_count + other.sample_count, v)


def stats_of(act, channel_shape, keep_values=False) -> CalibStats:
    a = np.abs(np.asarray(act, np.float32)).reshape((-1,) + tuple(channel_shape))
    return CalibStats(a.max(axis=0) if a.shape[0] else np.zeros(channel_shape, np.float32), a.shape[0],
                      np.sort(a.reshape(-1)) if keep_values else None)


@dataclass
class ClusterMap:
    """SPEC.md:371-377."""
    head_perm: np.ndarray                 # [nh] new position -> old head
    channel_perm: np.ndarray              # [nh, P] per OLD head: sorted position -> old channel
    head_group_bounds: np.ndarray         # [m+1]
    channel_group_bounds: np.ndarray      # [m, n+1]
    scales: np.ndarray                    # [m, n]

    @property
    def m(self):
        return len(self.head_group_bounds) - 1

    @property
    def n(self):
        return self.channel_group_bounds.shape[1] - 1

    def cell_of_new(self) -> np.ndarray:
        """Cell index (i*n + j) of every channel in the REORDERED layout [nh*P]."""
        nh, P = self.channel_perm.shape
        cells = np.empty(nh * P, np.int32)
        for i in range(self.m):
            for hp in range(self.head_group_bounds[i], self.head_group_bounds[i + 1]):
                for j in range(self.n):
                    lo, hi = self.channel_group_bounds[i, j], self.channel_group_bounds[i, j + 1]
                    cells[hp * P + lo:hp * P + hi] = i * self.n + j
        return cells


@dataclass
class StateGroupScales:
    """SPEC.md:378-381."""
    boundaries: np.ndarray
    scales_B: np.ndarray
    scales_C: np.ndarray
    scales_state: np.ndarray | None = None   # [m, n] over ClusterMap cells
    extra: dict = field(default_factory=dict)


def _sqdist(x, c):
    return ((x - c) ** 2).sum()


def kmeans(X, k: int, seed: int = 0, iters: int = 100) -> np.ndarray:
    """Literal Lloyd k-means with k-means++ init; returns labels [n]."""
    X = np.asarray(X, np.float64)
    n = X.shape[0]
    rng = make_rng(seed, KMEANS_STREAM)
    first = int(rng.integers(n))
    centers = [X[first].copy()]
    for _ in range(1, k):
        d2 = np.array([min(_sqdist(X[i], c) for c in centers) for i in range(n)])
        tot = d2.sum()
        if tot <= 0:
            centers.append(X[first].copy())
            continue
        r = rng.random() * tot
        idx = int(np.searchsorted(np.cumsum(d2), r, side="right"))
        centers.append(X[min(idx, n - 1)].copy())
    C = np.array(centers)
    labels = np.full(n, -1)
    for _ in range(iters):
        new = np.array([int(np.argmin([_sqdist(X[i], C[j]) for j in range(k)])) for i in range(n)])
        if np.array_equal(new, labels):
            break
        labels = new
        for j in range(k):
            mem = labels == j
            if mem.any():
                C[j] = X[mem].mean(axis=0)
    return labels


def _equal_groups(count: int, k: int) -> np.ndarray:
    return np.array([(i * k) // count for i in range(count)])


def sort_and_cluster(stats_x: CalibStats, n_heads: int, head_dim: int, m: int = 4, n: int = 4,
                     seed: int = 0, bits: int = 8) -> ClusterMap:
    """SPEC.md:393-401."""
    mx = np.asarray(stats_x.channel_max, np.float32).reshape(n_heads, head_dim)
    m = min(m, n_heads)
    n = min(n, head_dim)
    cperm = np.stack([np.argsort(-mx[h], kind="stable") for h in range(n_heads)]).astype(np.int64)
    F = np.stack([mx[h][cperm[h]] for h in range(n_heads)])
    if len(np.unique(F, axis=0)) < m:
        labels = _equal_groups(n_heads, m)
    else:
        labels = kmeans(F, m, seed)
    order = sorted(set(labels.tolist()), key=lambda l: int(np.min(np.nonzero(labels == l)[0])))
    head_perm = np.concatenate([np.nonzero(labels == l)[0] for l in order]).astype(np.int64)
    sizes = [int((labels == l).sum()) for l in order]
    hb = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    m_eff = len(order)
    cb = np.zeros((m_eff, n + 1), np.int64)
    scales = np.zeros((m_eff, n), np.float32)
    for i in range(m_eff):
        heads = head_perm[hb[i]:hb[i + 1]]
        v = F[heads].max(axis=0)
        if len(np.unique(v)) < n:
            lab = _equal_groups(head_dim, n)
        else:
            lab = kmeans(v[:, None], n, seed)
        cuts = [p for p in range(1, head_dim) if lab[p] != lab[p - 1]]
        if len(cuts) != n - 1:
            lab = _equal_groups(head_dim, n)
            cuts = [p for p in range(1, head_dim) if lab[p] != lab[p - 1]]
        cb[i] = [0] + cuts + [head_dim]
        for j in range(n):
            scales[i, j] = compute_scale(F[heads][:, cb[i, j]:cb[i, j + 1]], bits)
    return ClusterMap(head_perm, cperm, hb, cb, scales)


def build_state_group_scales(stats_B: CalibStats, stats_C: CalibStats, n_state_groups: int, d_state: int,
                             stats_h: CalibStats | None = None, cmap: ClusterMap | None = None,
                             bits: int = 8) -> StateGroupScales:
    """SPEC.md:402-410 (+ cached-state scales over the ClusterMap cells, LEDGER G7)."""
    mb = np.asarray(stats_B.channel_max, np.float32).reshape(n_state_groups, d_state)
    mc = np.asarray(stats_C.channel_max, np.float32).reshape(n_state_groups, d_state)
    sB = np.array([compute_scale(mb[g], bits) for g in range(n_state_groups)], np.float32)
    sC = np.array([compute_scale(mc[g], bits) for g in range(n_state_groups)], np.float32)
    ss = None
    if stats_h is not None and cmap is not None:
        nh, P = cmap.channel_perm.shape
        hm = np.asarray(stats_h.channel_max, np.float32).reshape(nh, P)
        # reordered layout: new (h', p') <- old (head_perm[h'], channel_perm[head_perm[h']][p'])
        hm_new = np.stack([hm[cmap.head_perm[hp]][cmap.channel_perm[cmap.head_perm[hp]]] for hp in range(nh)])
        cells = cmap.cell_of_new().reshape(nh, P)
        ss = np.ones((cmap.m, cmap.n), np.float32)
        for i in range(cmap.m):
            for j in range(cmap.n):
                ss[i, j] = compute_scale(hm_new[cells == i * cmap.n + j], bits)
    bnd = np.arange(n_state_groups + 1) * d_state
    return StateGroupScales(bnd, sB, sC, ss)


def calibrate_site_scale(stats: CalibStats, bits: int = 8, clip_percentile=None) -> np.float32:
    """SPEC.md:411-419."""
    if clip_percentile is not None and stats.values is not None and stats.values.size:
        return compute_scale(stats.values, bits, clip_percentile)
    return compute_scale(stats.channel_max, bits)
