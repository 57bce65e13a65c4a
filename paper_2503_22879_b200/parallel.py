"""Head-shard tensor parallelism for the Mamba2 block (the optional mode beside the
primary batch-shard replicas of ``dist``).  PAPER.md:174: Mamba2 computes (x, B, C, Δ) with one
projection "so the block is friendly to tensor parallelism".

Rank r of W owns heads [r·nh/W, (r+1)·nh/W): their rows of in_proj (z, x, Δ slices), the state
groups those heads read (B, C rows; a group shared by several shards is replicated), their conv
channels, SSM parameters, cached state, norm weight, and the matching K-slice of out_proj
(row-parallel).  conv, scan / SSD, gated norm, Hadamard and quant stay shard-local, so the only
collective is one all-reduce (sum) of the out_proj partials per layer — over NCCL / NVLink when
the block runs under torchrun.

That needs the model recipe to be shard-local: the gated RMSNorm runs over groups of
d_inner/W channels and the online Hadamard over blocks inside a group (``Dims.norm_groups`` = W,
``Dims.had_block``), mirrored in the oracle (oracle/ssm_block.py rmsnorm(groups), oracle/qblock.py)
and in the offline out_proj Hadamard fusion.  With norm_groups = 1 (the SPEC recipe) the norm and
FWHT span all heads and only batch sharding applies.
"""
from __future__ import annotations

from dataclasses import replace

import numpy as np
import torch

from .errors import ShapeError
from .ssm_block import DeviceBlock, Dims, QBlock, QLinear

__all__ = ["shard_qblock", "HeadShardedBlock"]


def _rows(ql: QLinear | None, idx: np.ndarray) -> QLinear | None:
    if ql is None:
        return None
    return QLinear(ql.kind, np.asarray(ql.codes)[idx], None if ql.s_ch is None else np.asarray(ql.s_ch)[idx],
                   None if ql.s_group is None else np.asarray(ql.s_group)[idx], ql.group)


def _cols(ql: QLinear, lo: int, hi: int) -> QLinear:
    """K-slice [lo, hi) of a projection: exact for per-row scales (W8) and for per-group scales
    when the slice is group-aligned (W4)."""
    codes = np.asarray(ql.codes)[:, lo:hi]
    if ql.s_group is not None:
        if lo % ql.group or hi % ql.group:
            raise ShapeError(f"K-slice [{lo},{hi}) is not aligned to the {ql.group}-wide quant groups")
        sg = np.asarray(ql.s_group)[:, lo // ql.group:hi // ql.group]
        return QLinear(ql.kind, codes, None, sg, ql.group)
    return QLinear(ql.kind, codes, None if ql.s_ch is None else np.asarray(ql.s_ch), None, ql.group)


def shard_qblock(qb: QBlock, world: int, rank: int) -> QBlock:
    """The rank's head shard of a quantized Mamba2 block (weights, scales and tables sliced; the
    result is an ordinary QBlock that runs on the same kernels)."""
    d = qb.dims
    if d.variant != "mamba2":
        raise ShapeError("head sharding applies to Mamba2 blocks")
    if d.n_heads % world or not 0 <= rank < world:
        raise ShapeError(f"{d.n_heads} heads do not split over {world} ranks")
    if d.norm_groups != world:
        raise ShapeError(f"head shards need the shard-local recipe (norm_groups == {world}, got {d.norm_groups})")
    nh, P, N, di = d.n_heads, d.head_dim, d.d_state, d.d_inner
    hs = nh // world
    h0, h1 = rank * hs, (rank + 1) * hs
    x_idx = np.arange(h0 * P, h1 * P)
    hg = np.asarray(qb.head_group, np.int64)
    groups = np.unique(hg[h0:h1])                       # state groups read by the shard's heads
    local = {int(g): i for i, g in enumerate(groups)}
    gn = d.n_state_groups * N
    b_idx = np.concatenate([np.arange(g * N, (g + 1) * N) for g in groups])
    in_rows = np.concatenate([x_idx, di + x_idx, 2 * di + b_idx, 2 * di + gn + b_idx, 2 * di + 2 * gn + np.arange(h0, h1)])
    conv_rows = np.concatenate([x_idx, di + b_idx, di + gn + b_idx])
    ld = Dims("mamba2", d.d_model, hs * P, N, hs, P, len(groups), d.conv_kernel, 0, 1)
    take = lambda a, idx: None if a is None else np.asarray(a)[idx]   # noqa: E731
    return replace(qb, dims=ld, in_proj=_rows(qb.in_proj, in_rows), out_proj=_cols(qb.out_proj, h0 * P, h1 * P),
                   conv_weight=take(qb.conv_weight, conv_rows), conv_bias=take(qb.conv_bias, conv_rows),
                   a_log=take(qb.a_log, np.arange(h0, h1)), d_param=take(qb.d_param, np.arange(h0, h1)),
                   dt_bias=take(qb.dt_bias, np.arange(h0, h1)), norm_weight=take(qb.norm_weight, x_idx),
                   head_group=np.array([local[int(g)] for g in hg[h0:h1]], np.int32),
                   in_out_scale=take(qb.in_out_scale, in_rows), conv_in_scale=take(qb.conv_in_scale, conv_rows),
                   conv_out_scale=take(qb.conv_out_scale, conv_rows), state_scale=take(qb.state_scale, x_idx),
                   extra=dict(qb.extra, shard=(rank, world)))


class HeadShardedBlock:
    """One rank's shard of a block on its GPU.  ``forward_codes`` returns the all-reduced block
    output: the local out_proj partial (f32 [B·T × d_model]) summed over the ranks by
    ``torch.distributed.all_reduce`` (NCCL on GPUs), the block's only collective."""

    def __init__(self, qb: QBlock, world: int, rank: int, dev="cuda", group=None):
        self.world, self.rank, self.group = world, rank, group
        self.local = DeviceBlock(shard_qblock(qb, world, rank), dev)
        self.dims = self.local.dims

    def new_state(self, batch: int, dev="cuda"):
        return self.local.new_state(batch, dev)

    def forward_codes(self, u_codes, B, T, state, state_in, out=None):
        part = self.local.forward_codes(u_codes, B, T, state, state_in, ws={"out": out} if out is not None else None)
        if self.world > 1:
            torch.distributed.all_reduce(part, op=torch.distributed.ReduceOp.SUM, group=self.group)
        return part
