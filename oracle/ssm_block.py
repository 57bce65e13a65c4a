"""Oracle: SPEC `[MODULE] ssm_block` float path.

TEST INFRASTRUCTURE ONLY.

Layout conventions (LEDGER G4):
* weights are [out × in]; y = u · Wᵀ.
* Mamba2 in_proj rows: z | x | B | C | Δ  (d_inner, d_inner, G·N, G·N, nh).
* Mamba1 in_proj rows: z | x (d_inner each); x_proj rows Δ_low | B | C
  (R, N, N); dt_proj [d_inner × R].
* SsmState.h is [n_heads × head_dim × d_state] (Mamba1: n_heads=1,
  head_dim=d_inner); conv_cache is [channels × (kernel-1)].
* ``head_group[h]`` names the state group of head h; it is h // (nh/G) until a
  head permutation is applied (reorder keeps B/C untouched).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from oracle.tensor_core import matmul, matmul_fast

EPS_NORM = np.float32(1e-5)


@dataclass
class Dims:
    variant: str              # "mamba2" | "mamba1"
    d_model: int
    d_inner: int
    d_state: int
    n_heads: int
    head_dim: int
    n_state_groups: int
    conv_kernel: int = 4
    dt_rank: int = 0          # Mamba1 only
    norm_groups: int = 1      # gated RMSNorm groups (1 = full d_inner; LEDGER G13)

    @property
    def had_block(self):
        """Online Hadamard block (LEDGER G9): largest power of two dividing d_inner / norm_groups,
        so no block crosses a norm group (head-shard recipe)."""
        g = self.d_inner // self.norm_groups
        return g & (-g)

    @property
    def conv_dim(self):
        if self.variant == "mamba2":
            return self.d_inner + 2 * self.n_state_groups * self.d_state
        return self.d_inner

    @property
    def in_proj_out(self):
        if self.variant == "mamba2":
            return 2 * self.d_inner + 2 * self.n_state_groups * self.d_state + self.n_heads
        return 2 * self.d_inner


@dataclass
class SsmBlockWeights:
    """SPEC.md:260-265 (+ Mamba1 x_proj/dt_proj, LEDGER G4)."""
    dims: Dims
    in_proj: np.ndarray
    conv_weight: np.ndarray
    conv_bias: np.ndarray
    a_log: np.ndarray
    d_param: np.ndarray
    dt_bias: np.ndarray
    norm_weight: np.ndarray
    out_proj: np.ndarray
    x_proj: np.ndarray | None = None
    dt_proj: np.ndarray | None = None
    head_group: np.ndarray | None = None
    applied: tuple = ()

    def __post_init__(self):
        d = self.dims
        if self.head_group is None and d.variant == "mamba2":
            self.head_group = (np.arange(d.n_heads) // (d.n_heads // d.n_state_groups)).astype(np.int32)

    @property
    def A(self):
        return (-np.exp(self.a_log.astype(np.float32))).astype(np.float32)

    def copy(self, **kw):
        return replace(self, **kw)


@dataclass
class SsmState:
    """SPEC.md:266-269."""
    h: np.ndarray
    conv_cache: np.ndarray
    extra: dict = field(default_factory=dict)


def zero_state(d: Dims) -> SsmState:
    if d.variant == "mamba2":
        h = np.zeros((d.n_heads, d.head_dim, d.d_state), np.float32)
    else:
        h = np.zeros((1, d.d_inner, d.d_state), np.float32)
    return SsmState(h, np.zeros((d.conv_dim, d.conv_kernel - 1), np.float32))


def silu(v):
    v = np.asarray(v, np.float32)
    with np.errstate(over="ignore"):   # exp(-v) = inf for v << 0: silu -> -0, the right limit
        return (v / (np.float32(1.0) + np.exp(-v))).astype(np.float32)


def softplus(v):
    """LEDGER G14: log1p(exp(x)), identity for x > 20."""
    v = np.asarray(v, np.float32)
    with np.errstate(over="ignore"):
        sp = np.log1p(np.exp(v)).astype(np.float32)
    return np.where(v > np.float32(20.0), v, sp).astype(np.float32)


def _gemm(a, w, fast):
    return (matmul_fast if fast else matmul)(a, np.ascontiguousarray(np.asarray(w, np.float32).T))


def project_inputs(u, w: SsmBlockWeights, fast=False):
    """SPEC.md:272-280.  Mamba2 → (x, B, C, Δ_raw, z) with xBC pre-conv;
    Mamba1 → (x, None, None, None, z) (B/C/Δ come from x_proj after conv)."""
    d = w.dims
    zx = _gemm(np.asarray(u, np.float32), w.in_proj, fast)
    di = d.d_inner
    z = zx[:, :di]
    x = zx[:, di:2 * di]
    if d.variant == "mamba1":
        return x, None, None, None, z
    gn = d.n_state_groups * d.d_state
    B = zx[:, 2 * di:2 * di + gn]
    C = zx[:, 2 * di + gn:2 * di + 2 * gn]
    dt = zx[:, 2 * di + 2 * gn:]
    return x, B, C, dt, z


def project_ssm_params(x_conv, w: SsmBlockWeights, fast=False):
    """Mamba1 sequential projections F_Δ = Proj(Proj(x))."""
    d = w.dims
    xd = _gemm(x_conv, w.x_proj, fast)
    R, N = d.dt_rank, d.d_state
    dt_low, B, C = xd[:, :R], xd[:, R:R + N], xd[:, R + N:R + 2 * N]
    dt = _gemm(dt_low, w.dt_proj, fast)
    return dt, B, C, dt_low


def causal_conv1d(x, weight, bias, cache=None):
    """depthwise causal conv + SiLU; returns (y, new_cache).
    acc = bias; acc += w[c,j]·x[t-K+1+j] for j ascending (f32, unfused)."""
    x = np.asarray(x, np.float32)
    wt = np.asarray(weight, np.float32)
    T, Cc = x.shape
    K = wt.shape[1]
    if cache is None:
        cache = np.zeros((Cc, K - 1), np.float32)
    if cache.shape != (Cc, K - 1):
        from oracle.errors import ShapeError
        raise ShapeError("cache/channel mismatch")
    xpad = np.concatenate([np.asarray(cache, np.float32).T, x], axis=0)
    acc = np.broadcast_to(np.asarray(bias, np.float32), (T, Cc)).astype(np.float32)
    for j in range(K):
        acc = (acc + (wt[:, j][None, :] * xpad[j:j + T]).astype(np.float32)).astype(np.float32)
    new_cache = np.ascontiguousarray(xpad[xpad.shape[0] - (K - 1):].T) if K > 1 else np.zeros((Cc, 0), np.float32)
    return silu(acc), new_cache


def discretize(dt_raw, dt_bias, A):
    """Δ = softplus(Δ_raw + dt_bias); Ȧ = exp(Δ·A).
    Mamba2: Δ [T×nh], A [nh]; Mamba1: Δ [T×d], A [d×N] → Ȧ [T×d×N]."""
    dt = softplus(np.asarray(dt_raw, np.float32) + np.asarray(dt_bias, np.float32))
    A = np.asarray(A, np.float32)
    if A.ndim == 1:
        dA = np.exp((dt * A[None, :]).astype(np.float32)).astype(np.float32)
    else:
        dA = np.exp((dt[:, :, None] * A[None, :, :]).astype(np.float32)).astype(np.float32)
    return dA, dt


def selective_scan(x, dA, dt, B, C, D, z=None, state=None, head_group=None, hmax=None):
    """SPEC.md:299-307, Eq. 2: h_t = Ȧ_t h_{t-1} + (Δ_t x_t) B_t; y_t = C_t·h_t + D x_t;
    optional gate y·SiLU(z).  Mamba2 when x is [T×nh×P] (B/C [T×G×N]);
    Mamba1 when x is [T×d] (Ȧ [T×d×N], B/C [T×N]).  Returns (y, h).
    ``hmax`` (a dict) receives max_t,n |h_t| per (head, channel) for state
    calibration (StateGroupScales)."""
    x = np.asarray(x, np.float32)
    T = x.shape[0]
    if x.ndim == 3:
        _, nh, P = x.shape
        G, N = B.shape[1], B.shape[2]
        hg = np.asarray(head_group) if head_group is not None else np.arange(nh) // (nh // G)
        h = np.zeros((nh, P, N), np.float32) if state is None else np.array(state, np.float32)
        y = np.empty((T, nh, P), np.float32)
        for t in range(T):
            Bt = B[t][hg]          # [nh, N]
            Ct = C[t][hg]
            dtx = (dt[t][:, None] * x[t]).astype(np.float32)            # [nh, P]
            h = (dA[t][:, None, None] * h + (dtx[:, :, None] * Bt[:, None, :]).astype(np.float32)).astype(np.float32)
            y[t] = (np.einsum("hpn,hn->hp", h.astype(np.float64), Ct.astype(np.float64)).astype(np.float32)
                    + (np.asarray(D, np.float32)[:, None] * x[t]).astype(np.float32))
            if hmax is not None:
                m = np.abs(h).max(axis=2)
                hmax["h"] = m if "h" not in hmax else np.maximum(hmax["h"], m)
    else:
        _, d = x.shape
        N = B.shape[1]
        h = np.zeros((d, N), np.float32) if state is None else np.array(state, np.float32).reshape(d, N)
        y = np.empty((T, d), np.float32)
        for t in range(T):
            dtx = (dt[t] * x[t]).astype(np.float32)
            h = (dA[t] * h + (dtx[:, None] * B[t][None, :]).astype(np.float32)).astype(np.float32)
            y[t] = (h.astype(np.float64) @ C[t].astype(np.float64)).astype(np.float32) + (np.asarray(D, np.float32) * x[t])
            if hmax is not None:
                m = np.abs(h).max(axis=1)[None, :]
                hmax["h"] = m if "h" not in hmax else np.maximum(hmax["h"], m)
        h = h.reshape(1, d, N)
    if z is not None:
        y = (y * silu(np.asarray(z, np.float32).reshape(y.shape))).astype(np.float32)
    return y, h


def ssd_chunked(x, dA, dt, B, C, D, z=None, chunk=64, state=None, head_group=None):
    """chunked SSD (intra-chunk (L∘CBᵀ)X + inter-chunk carry),
    float64 internally.  Mamba2 shapes only."""
    if chunk < 1:
        raise ValueError("chunk must be >= 1")
    x = np.asarray(x, np.float64)
    T, nh, P = x.shape
    G, N = B.shape[1], B.shape[2]
    hg = np.asarray(head_group) if head_group is not None else np.arange(nh) // (nh // G)
    la = np.log(np.asarray(dA, np.float64))                 # Δ·A
    dt = np.asarray(dt, np.float64)
    Bh = np.asarray(B, np.float64)[:, hg]                   # [T, nh, N]
    Ch = np.asarray(C, np.float64)[:, hg]
    H = np.zeros((nh, P, N)) if state is None else np.array(state, np.float64)
    y = np.empty((T, nh, P))
    for t0 in range(0, T, chunk):
        t1 = min(T, t0 + chunk)
        cs = np.cumsum(la[t0:t1], axis=0)                   # [Q, nh]
        Q = t1 - t0
        seg = cs[:, None, :] - cs[None, :, :]               # [t, s, nh]
        mask = np.tril(np.ones((Q, Q), bool))
        L = np.where(mask[:, :, None], np.exp(np.where(mask[:, :, None], seg, 0.0)), 0.0)
        CB = np.einsum("thn,shn->tsh", Ch[t0:t1], Bh[t0:t1])
        W = CB * L * dt[t0:t1][None, :, :]                  # [t, s, nh]
        ydiag = np.einsum("tsh,shp->thp", W, x[t0:t1])
        yoff = np.exp(cs)[:, :, None] * np.einsum("thn,hpn->thp", Ch[t0:t1], H)
        y[t0:t1] = ydiag + yoff + np.asarray(D, np.float64)[None, :, None] * x[t0:t1]
        decay = np.exp(cs[-1][None, :] - cs)                # [Q, nh]
        H = np.exp(cs[-1])[:, None, None] * H + np.einsum("sh,shp,shn->hpn", decay * dt[t0:t1], x[t0:t1], Bh[t0:t1])
    y = y.astype(np.float32)
    if z is not None:
        y = (y * silu(np.asarray(z, np.float32).reshape(y.shape))).astype(np.float32)
    return y, H.astype(np.float32)


def rmsnorm(v, weight, eps=EPS_NORM, groups: int = 1):
    """RMS normalisation over the last axis (full d_inner, LEDGER G13), or over
    ``groups`` contiguous equal slices of it (the grouped norm of the head-shard recipe)."""
    v = np.asarray(v, np.float32)
    if groups > 1:
        n = v.shape[-1]
        vg = v.reshape(v.shape[:-1] + (groups, n // groups))
        ms = np.mean(vg.astype(np.float64) ** 2, axis=-1, keepdims=True).astype(np.float32)
        r = (np.float32(1.0) / np.sqrt(ms + np.float32(eps))).astype(np.float32)
        return ((vg * r).astype(np.float32).reshape(v.shape) * np.asarray(weight, np.float32)).astype(np.float32)
    ms = np.mean(v.astype(np.float64) ** 2, axis=-1, keepdims=True).astype(np.float32)
    r = (np.float32(1.0) / np.sqrt(ms + np.float32(eps))).astype(np.float32)
    return ((v * r).astype(np.float32) * np.asarray(weight, np.float32)).astype(np.float32)


def block_forward_float(u, w: SsmBlockWeights, state: SsmState | None = None, chunk=None,
                        fast=False, taps: dict | None = None):
    """project → conv → discretize → scan/SSD → gate → norm →
    out_proj.  Returns (out [T×d_model], new SsmState).  ``taps`` (if given)
    receives the calibration sites."""
    d = w.dims
    u = np.asarray(u, np.float32)
    st = state if state is not None else zero_state(d)
    x, B, C, dt_raw, z = project_inputs(u, w, fast)
    if d.variant == "mamba2":
        xBC = np.concatenate([x, B, C], axis=1)
        conv_out, cache = causal_conv1d(xBC, w.conv_weight, w.conv_bias, st.conv_cache)
        di, gn = d.d_inner, d.n_state_groups * d.d_state
        xc = conv_out[:, :di]
        Bc = conv_out[:, di:di + gn].reshape(-1, d.n_state_groups, d.d_state)
        Cc = conv_out[:, di + gn:].reshape(-1, d.n_state_groups, d.d_state)
        dA, dt = discretize(dt_raw, w.dt_bias, w.A)
        xh = xc.reshape(-1, d.n_heads, d.head_dim)
        zh = z.reshape(-1, d.n_heads, d.head_dim)
        hm = {} if taps is not None else None
        if chunk is None or taps is not None:
            y, h = selective_scan(xh, dA, dt, Bc, Cc, w.d_param, zh, st.h, w.head_group, hmax=hm)
        else:
            y, h = ssd_chunked(xh, dA, dt, Bc, Cc, w.d_param, zh, chunk, st.h, w.head_group)
        y = y.reshape(-1, d.d_inner)
        if taps is not None:
            taps.update(u=u, z=z, x_in=x, B_in=B, C_in=C, dt=dt_raw, x=xc, B=Bc, C=Cc, h=hm["h"])
    else:
        xc, cache = causal_conv1d(x, w.conv_weight, w.conv_bias, st.conv_cache)
        dt_raw, B, C, dt_low = project_ssm_params(xc, w, fast)
        dA, dt = discretize(dt_raw, w.dt_bias, w.A)
        hm = {} if taps is not None else None
        y, h = selective_scan(xc, dA, dt, B, C, w.d_param, z, st.h, hmax=hm)
        if taps is not None:
            taps.update(u=u, z=z, x_in=x, x=xc, dt_low=dt_low, B=B, C=C, dt=dt_raw, h=hm["h"])
    r = rmsnorm(y, w.norm_weight, groups=d.norm_groups)
    if taps is not None:
        from oracle.hadamard import fwht_blocked
        taps.update(y=y, r=r, y_had=fwht_blocked(r, d.had_block))
    out = _gemm(r, w.out_proj, fast)
    return out, SsmState(h, cache)
