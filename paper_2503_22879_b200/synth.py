"""Synthetic random-init quantized models at the BASELINE shapes (no checkpoints exist
offline; BASELINE.json `data: synthetic`).

* ``random_qblock``  — host QBlock with analytic scales (parity tests at full shapes).
* ``device_qblock`` / ``synthetic_lm`` — weights generated directly in HBM (random int4
  bytes are valid nibble pairs), for the bench: a 56-layer 8B-shaped model is built in
  seconds without a host round trip.
Scales are chosen so every activation site uses most of its int8 range.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .ssm_block import DeviceBlock, Dims, QBlock, QLinear
from .tensor import make_rng

U_STD_CODES = 127.0 / 4.0     # N(0,1) inputs quantized with s = 4/127


def _slice_scales(d: Dims):
    s = np.float32(4.0 / 127)
    return s


def _analytic_qlinear(r, n, k, kind, group, out_std, in_code_std, s_a=1.0):
    """Weights whose outputs have std ~out_std (float units) for A8 inputs of code std
    in_code_std and input scale s_a (the epilogue multiplies by s_a), or float inputs of std 1."""
    group = min(group, k)
    if kind == "w8":
        codes = r.integers(-127, 128, (n, k)).astype(np.int8)
        rms = np.sqrt((codes.astype(np.float64) ** 2).mean(axis=1))
        s_ch = (out_std / (s_a * np.sqrt(k) * in_code_std * rms)).astype(np.float32)
        return QLinear("w8", codes, s_ch=s_ch, group=k)
    codes = r.integers(-8, 8, (n, k)).astype(np.int8)
    # per-group float scales (SPEC PerGroup); A8 inputs are codes of std in_code_std
    std_in = in_code_std * s_a if kind == "w4a8" else 1.0
    s_group = r.uniform(0.5, 1.5, (n, k // group)).astype(np.float32) * np.float32(out_std / (np.sqrt(k) * 4.6 * std_in))
    return QLinear(kind, codes, s_group=s_group.astype(np.float32), group=group)


def random_qblock(d: Dims, profile: str, seed: int = 0) -> QBlock:
    r = make_rng(seed, 11, 0)
    kind = {"W8A8": "w8", "W4A8": "w4a8", "W4A16": "w4a16"}[profile]
    di = d.d_inner
    s = np.float32(4.0 / 127)
    hb = d.had_block
    s_y = np.float32(4.5 * np.sqrt(hb) / 127)
    inp = _analytic_qlinear(r, d.in_proj_out, d.d_model, kind, 128, 1.0, U_STD_CODES, s)
    out = _analytic_qlinear(r, d.d_model, di, kind, 128, 0.1, 127.0 / 4.0, s_y)
    C = d.conv_dim
    K = d.conv_kernel
    conv_w = (r.standard_normal((C, K)) * 0.5 / np.sqrt(K)).astype(np.float32)
    conv_b = (r.standard_normal(C) * 0.05).astype(np.float32)
    nd = d.n_heads if d.variant == "mamba2" else di
    dtv = r.uniform(1e-3, 1e-1, nd)
    dt_bias = (dtv + np.log(-np.expm1(-dtv))).astype(np.float32)
    if d.variant == "mamba2":
        a_log = np.log(r.uniform(1, 16, d.n_heads)).astype(np.float32)
    else:
        a_log = np.log(np.tile(np.arange(1, d.d_state + 1, dtype=np.float32), (di, 1))).astype(np.float32)
    dpar = np.ones(nd, np.float32)
    norm = (1.0 + 0.1 * r.standard_normal(di)).astype(np.float32)
    qb = QBlock(d, profile, inp, out, conv_w, conv_b, a_log, dpar, dt_bias, norm,
                head_group=(np.arange(d.n_heads) // max(1, d.n_heads // d.n_state_groups)).astype(np.int32)
                if d.variant == "mamba2" else None,
                s_u=s, s_y=s_y)
    if profile == "W4A16":
        return qb
    qb.in_out_scale = np.full(d.in_proj_out, s, np.float32)
    qb.conv_in_scale = np.full(C, s, np.float32)
    qb.conv_out_scale = (r.uniform(0.5, 1.0, C) * 2.0 / 127).astype(np.float32)
    if d.variant == "mamba2":
        gn = d.n_state_groups * d.d_state
        qb.conv_out_scale[di:di + gn] = np.repeat(qb.conv_out_scale[di:di + gn:d.d_state], d.d_state)
        qb.conv_out_scale[di + gn:] = np.repeat(qb.conv_out_scale[di + gn::d.d_state], d.d_state)
        rows = d.n_heads * d.head_dim
    else:
        rows = di
        R, N = d.dt_rank, d.d_state
        qb.x_proj = _analytic_qlinear(r, R + 2 * N, di, "w8" if kind == "w8" else "w4a8", 128, 1.0, 64.0)
        qb.dt_proj = _analytic_qlinear(r, di, R, "w8" if kind == "w8" else "w4a8", 32, 1.0, U_STD_CODES, s)
        qb.xproj_out_scale = np.full(R + 2 * N, s, np.float32)
        qb.s_dt = s
    qb.state_scale = (r.uniform(0.5, 1.0, rows) * 0.5 / 127).astype(np.float32)
    return qb


@dataclass
class DeviceQL:
    """A projection whose kernel-layout weights are already in HBM."""
    kind: str
    shape: tuple
    group: int
    device_w: torch.Tensor
    s_ch: object = None
    s_group: object = None


def _device_ql(g: torch.Generator, n, k, kind, dev, group=128, in_code_std=U_STD_CODES, out_std=1.0, s_a=1.0):
    group = min(group, k)
    if kind == "w8":
        w = torch.randint(-127, 128, (n, k), generator=g, device=dev, dtype=torch.int8)
        s_ch = np.full(n, out_std / (s_a * np.sqrt(k) * in_code_std * 73.3), np.float32)
        return DeviceQL("w8", (n, k), k, w, s_ch=s_ch)
    from . import ops
    nbytes = ops.w4_bytes(n, k) if kind == "w4a8" else ops.w4a16_bytes(n, k, group)   # kernel layout
    w = torch.randint(0, 256, (nbytes,), generator=g, device=dev, dtype=torch.uint8)
    std_in = in_code_std * s_a if kind == "w4a8" else 1.0
    s_group = torch.rand((n, k // group), generator=g, device=dev, dtype=torch.float32).add_(0.5).mul_(
        out_std / (np.sqrt(k) * 4.6 * std_in))
    return DeviceQL(kind, (n, k), group, w, s_group=s_group)


def device_qblock(d: Dims, profile: str, seed: int, dev) -> DeviceBlock:
    """A DeviceBlock whose big projections are generated in HBM; small tensors on host."""
    kind = {"W8A8": "w8", "W4A8": "w4a8", "W4A16": "w4a16"}[profile]
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    small = random_qblock(Dims(d.variant, 32, d.d_inner, d.d_state, d.n_heads, d.head_dim, d.n_state_groups,
                               d.conv_kernel, d.dt_rank), profile, seed)
    small.dims = d
    small.in_proj = _device_ql(g, d.in_proj_out, d.d_model, kind, dev, s_a=small.s_u)
    small.out_proj = _device_ql(g, d.d_model, d.d_inner, kind, dev, in_code_std=127.0 / 4, out_std=0.1, s_a=small.s_y)
    if profile != "W4A16":
        small.in_out_scale = np.full(d.in_proj_out, np.float32(4.0 / 127), np.float32)
        if d.variant == "mamba1":
            R, N = d.dt_rank, d.d_state
            k2 = "w8" if kind == "w8" else "w4a8"
            small.x_proj = _device_ql(g, R + 2 * N, d.d_inner, k2, dev, in_code_std=64.0)
            small.dt_proj = _device_ql(g, d.d_inner, R, k2, dev, group=32, s_a=small.s_u)
    return DeviceBlock(small, dev)


@dataclass
class SynthHost:
    dims: Dims
    profiles: list
    emb_codes: object
    emb_scale: object
    layer_norms: list
    blocks: list
    final_norm: object
    head: object
    s_head: float


def head_shard_dims(d: Dims, world: int) -> Dims:
    """Block dims of one rank's head shard (parallel.shard_qblock's shape): nh/W heads, their
    d_inner/W channels and G/W state groups, the norm / Hadamard local to the shard."""
    if d.variant != "mamba2" or d.n_heads % world or d.n_state_groups % world:
        raise ValueError(f"{d.n_heads} heads / {d.n_state_groups} groups do not split over {world} ranks")
    return Dims("mamba2", d.d_model, d.d_inner // world, d.d_state, d.n_heads // world, d.head_dim,
                d.n_state_groups // world, d.conv_kernel)


def synthetic_lm(d: Dims, n_layers: int, profile: str, vocab: int, dev="cuda", seed: int = 0, head_kind="w4a8",
                 tp_group=None):
    """Random-init model in HBM.  With ``tp_group`` the blocks are this rank's head shards of
    ``d`` (head_shard_dims) and the model all-reduces their out_proj partials."""
    from .model import QuantizedMambaLM
    if tp_group is not None:
        d = head_shard_dims(d, torch.distributed.get_world_size(tp_group))
    g = torch.Generator(device=dev)
    g.manual_seed(seed + 1000)
    emb = torch.randint(-127, 128, (vocab, d.d_model), generator=g, device=dev, dtype=torch.int8)
    es = torch.full((vocab,), 1.0 / 127, device=dev)
    blocks = [device_qblock(d, profile, seed + l, dev) for l in range(n_layers)]
    head = _device_ql(g, vocab, d.d_model, head_kind, dev, s_a=np.float32(4.0 / 127))
    host = SynthHost(d, [profile] * n_layers, emb, es, [np.ones(d.d_model, np.float32)] * n_layers, blocks,
                     np.ones(d.d_model, np.float32), head, np.float32(4.0 / 127))
    return QuantizedMambaLM(host, dev, tp_group=tp_group)
