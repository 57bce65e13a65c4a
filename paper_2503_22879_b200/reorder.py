"""reorder — SPEC `[MODULE] reorder`: offline cluster-aware weight
rearrangement, so the runtime sees x already sorted/clustered and no
online permutation is needed.

π[h'·P + p'] = head_perm[h']·P + channel_perm[head_perm[h']][p']

Rewritten tensors:
* Mamba2: in_proj rows of z and x by π, Δ rows by head_perm; conv x channels by π;
  a_log, D, dt_bias by head_perm; norm weight by π; out_proj columns by π;
  head_group[h'] = head_group[head_perm[h']]  (B/C untouched).
* Mamba1 (one "head" of d_inner channels, LEDGER G12): in_proj z/x rows, conv, x_proj
  columns, dt_proj rows, dt_bias, a_log rows, D, norm and out_proj columns by π.
Reorder runs before Hadamard fusion.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import PipelineError, ShapeError

__all__ = ["ReorderPlan", "build_reorder_plan", "apply_reorder", "permute_state"]


@dataclass
class ReorderPlan:
    pi: np.ndarray
    head_perm: np.ndarray
    head_dim: int
    tag: str = "reorder"

    def inverse(self) -> "ReorderPlan":
        return ReorderPlan(np.argsort(self.pi), np.argsort(self.head_perm), self.head_dim, self.tag + "^-1")


def build_reorder_plan(cmap, dims) -> ReorderPlan:
    nh, P = (1, dims.d_inner) if dims.variant == "mamba1" else (dims.n_heads, dims.head_dim)
    hp = np.asarray(cmap.head_perm, np.int64)
    cp = np.asarray(cmap.channel_perm, np.int64)
    if cp.shape != (nh, P) or not np.array_equal(np.sort(hp), np.arange(nh)):
        raise ShapeError("ClusterMap inconsistent with the block dims")
    pi = (hp[:, None] * P + cp[hp]).reshape(-1)
    return ReorderPlan(pi, hp, P)


def apply_reorder(w, plan: ReorderPlan):
    """Returns a new SsmBlockWeights; refuses a plan already applied."""
    d = w.dims
    if plan.tag in w.applied:
        raise PipelineError("reorder plan already applied")
    di = d.d_inner
    pi, hp = np.asarray(plan.pi), np.asarray(plan.head_perm)
    if len(pi) != di:
        raise ShapeError("plan / d_inner mismatch")
    rows = np.arange(w.in_proj.shape[0])
    rows[:di] = pi
    rows[di:2 * di] = di + pi
    conv_rows = np.arange(w.conv_weight.shape[0])
    conv_rows[:di] = pi
    kw = dict(conv_weight=w.conv_weight[conv_rows].copy(), conv_bias=w.conv_bias[conv_rows].copy(),
              norm_weight=w.norm_weight[pi].copy(), out_proj=w.out_proj[:, pi].copy(),
              applied=tuple(w.applied) + (plan.tag,))
    if d.variant == "mamba2":
        base = 2 * di + 2 * d.n_state_groups * d.d_state
        rows[base:] = base + hp
        kw.update(in_proj=w.in_proj[rows].copy(), a_log=w.a_log[hp].copy(), d_param=w.d_param[hp].copy(),
                  dt_bias=w.dt_bias[hp].copy(), head_group=np.asarray(w.head_group)[hp].astype(np.int32))
    else:
        kw.update(in_proj=w.in_proj[rows].copy(), x_proj=w.x_proj[:, pi].copy(), dt_proj=w.dt_proj[pi].copy(),
                  dt_bias=w.dt_bias[pi].copy(), a_log=w.a_log[pi].copy(), d_param=w.d_param[pi].copy())
    return w.copy(**kw)


def permute_state(h, plan: ReorderPlan):
    """SsmState.h [nh × P × N] from the original to the reordered layout."""
    h = np.asarray(h)
    nh, P, N = h.shape
    return h.reshape(nh * P, N)[plan.pi].reshape(nh, P, N)
