"""Float reference block and model forward in torch, with the calibration
taps of SPEC.md:384-392.  Offline only: it feeds `calibrate.collect_stats` (the paper's
static abs-max calibration).  The quantized hot path never uses it.

Conventions as the block contract (ssm_block module docstring): weights [out × in]; Mamba2
in_proj rows z | x | B | C | Δ; Mamba1 in_proj rows z | x, x_proj rows Δ_low | B | C.
Projections run in float64 (exactly-rounded float32 results up to summation order), the
recurrence in float32 like the SPEC scan.
"""
from __future__ import annotations

import numpy as np
import torch

from .hadamard import fwht_blocked

EPS_NORM = 1e-5


def _t(a, dev, dt=torch.float32):
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dt)
    return torch.as_tensor(np.asarray(a)).to(device=dev, dtype=dt)


def _proj(a: torch.Tensor, w, dev) -> torch.Tensor:
    return (a.to(torch.float64) @ _t(w, dev, torch.float64).T).to(torch.float32)


def silu(v):
    return v / (1.0 + torch.exp(-v))


def softplus(v):
    return torch.where(v > 20.0, v, torch.log1p(torch.exp(torch.clamp(v, max=20.0))))


def rmsnorm(v, weight, groups: int = 1):
    if groups > 1:   # grouped norm (head-shard recipe): contiguous equal slices of the last axis
        vg = v.reshape(*v.shape[:-1], groups, v.shape[-1] // groups)
        ms = (vg.to(torch.float64) ** 2).mean(dim=-1, keepdim=True).to(torch.float32)
        return ((vg * (1.0 / torch.sqrt(ms + np.float32(EPS_NORM)))).reshape(v.shape)) * weight
    ms = (v.to(torch.float64) ** 2).mean(dim=-1, keepdim=True).to(torch.float32)
    r = 1.0 / torch.sqrt(ms + np.float32(EPS_NORM))
    return (v * r) * weight


def causal_conv1d(x, weight, bias):
    """SPEC.md:281-289 on a fresh cache: acc = bias + Σ_j w[c,j]·x[t-K+1+j] (j ascending)."""
    T, C = x.shape
    K = weight.shape[1]
    xp = torch.cat([torch.zeros((K - 1, C), dtype=x.dtype, device=x.device), x], 0)
    acc = bias.expand(T, C).clone()
    for j in range(K):
        acc = acc + weight[:, j][None, :] * xp[j:j + T]
    return silu(acc)


def block_forward_float(u, w, taps: dict | None = None, device="cuda"):
    """project -> conv -> discretize -> scan -> gate -> norm -> out_proj
    for one sequence u [T × d_model]; ``taps`` receives the calibration sites."""
    d = w.dims
    dev = torch.device(device)
    u = _t(u, dev)
    zx = _proj(u, w.in_proj, dev)
    di = d.d_inner
    z, x = zx[:, :di], zx[:, di:2 * di]
    conv_w, conv_b = _t(w.conv_weight, dev), _t(w.conv_bias, dev)
    dt_bias = _t(w.dt_bias, dev)
    A = -torch.exp(_t(w.a_log, dev))
    D = _t(w.d_param, dev)
    T = u.shape[0]
    if d.variant == "mamba2":
        gn = d.n_state_groups * d.d_state
        Bin, Cin, dt_raw = zx[:, 2 * di:2 * di + gn], zx[:, 2 * di + gn:2 * di + 2 * gn], zx[:, 2 * di + 2 * gn:]
        co = causal_conv1d(torch.cat([x, Bin, Cin], 1), conv_w, conv_b)
        xc = co[:, :di].reshape(T, d.n_heads, d.head_dim)
        Bc = co[:, di:di + gn].reshape(T, d.n_state_groups, d.d_state)
        Cc = co[:, di + gn:].reshape(T, d.n_state_groups, d.d_state)
        dt = softplus(dt_raw + dt_bias)
        dA = torch.exp(dt * A[None, :])
        hg = torch.as_tensor(np.asarray(w.head_group), dtype=torch.long, device=dev)
        h = torch.zeros((d.n_heads, d.head_dim, d.d_state), device=dev)
        hmax = torch.zeros((d.n_heads, d.head_dim), device=dev)
        ys = []
        for t in range(T):
            Bt, Ct = Bc[t][hg], Cc[t][hg]
            dtx = dt[t][:, None] * xc[t]
            h = dA[t][:, None, None] * h + dtx[:, :, None] * Bt[:, None, :]
            y_t = torch.einsum("hpn,hn->hp", h.double(), Ct.double()).float() + D[:, None] * xc[t]
            ys.append(y_t)
            hmax = torch.maximum(hmax, h.abs().amax(dim=2))
        y = torch.stack(ys) * silu(z.reshape(T, d.n_heads, d.head_dim))
        y = y.reshape(T, di)
        if taps is not None:
            taps.update(u=u, z=z, x_in=x, B_in=Bin, C_in=Cin, dt=dt_raw, x=co[:, :di], B=Bc, C=Cc, h=hmax)
    else:
        R, N = d.dt_rank, d.d_state
        xc = causal_conv1d(x, conv_w, conv_b)
        xd = _proj(xc, w.x_proj, dev)
        dt_low, Bm, Cm = xd[:, :R], xd[:, R:R + N], xd[:, R + N:R + 2 * N]
        dt_raw = _proj(dt_low, w.dt_proj, dev)
        dt = softplus(dt_raw + dt_bias)
        dA = torch.exp(dt[:, :, None] * A[None])
        h = torch.zeros((di, N), device=dev)
        hmax = torch.zeros((1, di), device=dev)
        ys = []
        for t in range(T):
            h = dA[t] * h + (dt[t] * xc[t])[:, None] * Bm[t][None, :]
            ys.append((h.double() @ Cm[t].double()).float() + D * xc[t])
            hmax = torch.maximum(hmax, h.abs().amax(dim=1)[None])
        y = torch.stack(ys) * silu(z)
        if taps is not None:
            taps.update(u=u, z=z, x_in=x, x=xc, dt_low=dt_low, B=Bm, C=Cm, dt=dt_raw, h=hmax)
    r = rmsnorm(y, _t(w.norm_weight, dev), d.norm_groups)
    if taps is not None:
        taps.update(y=y, r=r, y_had=fwht_blocked(r, d.had_block))
    return _proj(r, w.out_proj, dev)


def float_forward(model, tokens, taps: list | None = None, device="cuda"):
    """Pre-norm residual stack (LEDGER G8): h = E[tok]; h += block(rmsnorm(h)); logits =
    head(rmsnorm(h)).  ``taps`` receives one dict per block plus {"head_in"}."""
    dev = torch.device(device)
    tokens = np.asarray(tokens)
    h = _t(np.asarray(model.embedding)[tokens], dev)
    for l, blk in enumerate(model.blocks):
        u = rmsnorm(h, _t(model.layer_norms[l], dev))
        t = {} if taps is not None else None
        h = h + block_forward_float(u, blk, t, device)
        if taps is not None:
            taps.append(t)
    hf = rmsnorm(h, _t(model.final_norm, dev))
    if taps is not None:
        taps.append({"head_in": hf})
    return _proj(hf, model.head, dev)
