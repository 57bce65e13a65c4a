"""Oracle: quantized block forward / decode (Fig. 4).

TEST INFRASTRUCTURE ONLY.

This fixes, as a format contract mirrored by the GPU kernels, every rounding
step of the A8 path (LEDGER G5, G6, G11, G16):

  u_q   = rint(u / s_u)                                  per-tensor (G5)
  W8A8  : acc = Σ_k a_q[k]·w8[n,k] (int32, exact);  y = f32(acc) · f32(s_ch[n]·s_a)
  W4A8  : acc_g = Σ_{k∈g} a_q[k]·w4[n,k] (int32 per 128-group, exact);
          p = fma(s_w[n,g], f32(acc_g), p) over g ascending (f32, one rounding each, as the
          kernels' FFMA; with a K split over S CTAs each split starts from 0 and the S
          partials add in order);
          y = f32(p · s_a)                                  (LEDGER G11)
  codes = clamp(rint(y / s_col[n]))     in_proj slices z|x|B|C|Δ per-tensor (G16)
  conv  : v = f32(q)·s_in[c]; acc = bias; acc += w[c,j]·v_j (j asc); silu;
          rint(silu / s_out[c])  with s_out = clustered x cells | B/C per group
  scan  : x̂ = x_q·s_x[c], B̂/Ĉ = q·s_B/C[g], Δ = softplus(Δ_q·s_Δ + dt_bias) (G6),
          Ȧ = exp(ΔA); h fp32; y = C·h + D·x̂; y·SiLU(z_q·s_z)
  state : cached as rint(h / s_h[cell(h,p)]) between calls (G7)
  norm  : r = y·rsqrt(mean y² + 1e-5)·γ   (full d_inner, G13)
  had   : ȳ = rint(H_blk r / s_y)           (unnormalised Sylvester blocks, G9)
  out   : f32(acc)·f32(s_ch·s_y)

Mamba1: x_proj consumes clustered-scale x, so the per-channel activation scale
is folded into the x_proj weight columns before per-channel quantisation
(s_a = 1 in its epilogue).  W4A16 runs the float path with dequantised
per-group weights and float (fp32) state; its projections take bf16
activations (north_star (a): int4-weight x bf16-activation GEMV): x is rounded to
bf16 (RN-even) before the product, everything else stays f32.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from oracle import hadamard as had
from oracle.quantizer import quantize_codes, quantize_weight_w4_group, quantize_weight_w8
from oracle.ssm_block import (Dims, causal_conv1d, discretize, rmsnorm, selective_scan)
from oracle.tensor_core import int_gemm, matmul_fast


@dataclass
class QLinear:
    kind: str                      # "w8" | "w4a8" | "w4a16"
    codes: np.ndarray              # int8 [n_out, k] (4-bit values for w4*)
    s_ch: np.ndarray | None = None     # [n_out]      (w8)
    s_group: np.ndarray | None = None  # [n_out, k/g] (w4a8 / w4a16: SPEC PerGroup float scales)
    group: int = 128

    @property
    def n_out(self):
        return self.codes.shape[0]

    @property
    def k(self):
        return self.codes.shape[1]

    def dequant(self):
        n, k = self.codes.shape
        g = self.group
        if self.kind in ("w4a8", "w4a16"):
            return (self.codes.astype(np.float32).reshape(n, k // g, g) * self.s_group[:, :, None]).reshape(n, k)
        return (self.codes.astype(np.float32) * self.s_ch[:, None]).astype(np.float32)


def make_qlinear(w, kind: str, group: int = 128) -> QLinear:
    w = np.asarray(w, np.float32)
    group = min(group, w.shape[1])
    if kind == "w8":
        q = quantize_weight_w8(w)
        return QLinear("w8", q.payload, s_ch=q.extra["s_ch"], group=w.shape[1])
    if kind in ("w4a8", "w4a16"):
        q = quantize_weight_w4_group(w, group)
        return QLinear(kind, q.payload, s_group=q.extra["s_group"], group=group)
    raise ValueError(kind)


def group_partials(a_codes, ql: QLinear) -> np.ndarray:
    """Exact per-group int32 partials acc_g [G, M, N] of a W4A8 projection."""
    a = np.asarray(a_codes, np.int8)
    n, k = ql.codes.shape
    g = ql.group
    return np.stack([int_gemm(a[:, i * g:(i + 1) * g], ql.codes[:, i * g:(i + 1) * g].T) for i in range(k // g)])


def fma32(a, b, c) -> np.ndarray:
    """f32 fused multiply-add, round(a·b + c) once.  a·b of two f32 values is exact in the x87
    64-bit significand, and so is the sum unless c dominates a·b by > 2^18, where the extended
    rounding can no longer land on an f32 midpoint: the f32 result is the correctly rounded one."""
    ld = np.longdouble
    return (np.asarray(a, np.float32).astype(ld) * np.asarray(b, np.float32).astype(ld)
            + np.asarray(c, np.float32).astype(ld)).astype(np.float32)


def promote_groups(accg, s_group, s_a, splits: int = 1) -> np.ndarray:
    """W4A8 scale promotion (LEDGER G11): per split, p = fma(s_w, f32(acc_g), p) over ascending
    groups from 0; the split partials add in split order; y = f32(p·s_a).  Bit-exact
    restatement of the kernels (tcgen05 FFMA2 promotion and the mma.sync fallback)."""
    G = accg.shape[0]
    total = None
    for s in range(splits):
        p = np.zeros(accg.shape[1:], np.float32)
        for i in range(s * G // splits, (s + 1) * G // splits):
            p = fma32(s_group[None, :, i], accg[i].astype(np.float32), p)
        total = p if total is None else (total + p).astype(np.float32)
    return (total * np.float32(s_a)).astype(np.float32)


# K-split policy of the device under test, (M, N, K) -> splits (tests register the kernel's
# sq_gemm_w4a8_splits so block-level comparisons follow its summation order); default 1.
SPLITS_FN = None


def qlinear_a8(a_codes, ql: QLinear, s_a, splits: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """A8 projection; returns (y f32, acc int64).  W8A8: acc is the exact int32 GEMM over K.
    W4A8: acc is Σ_g acc_g (the int32 total, for kernel checks) and y the promoted sum."""
    a = np.asarray(a_codes, np.int8)
    if splits is None:
        splits = SPLITS_FN(a.shape[0], ql.codes.shape[0], ql.codes.shape[1]) if SPLITS_FN and ql.group == 128 else 1
    if ql.kind == "w8":
        acc = int_gemm(a, ql.codes.T)
        alpha = (ql.s_ch * np.float32(s_a)).astype(np.float32)
        return (acc.astype(np.float32) * alpha[None, :]).astype(np.float32), acc
    accg = group_partials(a, ql)
    return promote_groups(accg, ql.s_group, s_a, splits), accg.sum(axis=0)


def round_bf16(a) -> np.ndarray:
    """f32 -> bfloat16 (round to nearest even), returned as f32 (finite inputs)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def qlinear_a16(a, ql: QLinear) -> np.ndarray:
    """W4A16 projection: bf16(a) @ dequant(w).T with f32 accumulation."""
    return matmul_fast(round_bf16(a), ql.dequant().T)


@dataclass
class QBlock:
    """Quantized block weights + per-activation scale set (SPEC `plan`)."""
    dims: Dims
    profile: str                   # "W8A8" | "W4A8" | "W4A16"
    in_proj: QLinear
    out_proj: QLinear
    conv_weight: np.ndarray
    conv_bias: np.ndarray
    a_log: np.ndarray
    d_param: np.ndarray
    dt_bias: np.ndarray
    norm_weight: np.ndarray
    head_group: np.ndarray | None = None
    x_proj: QLinear | None = None
    dt_proj: QLinear | None = None
    # activation scales (A8 profiles)
    s_u: np.float32 = np.float32(1.0)
    in_out_scale: np.ndarray | None = None      # [in_proj_out]
    conv_in_scale: np.ndarray | None = None     # [conv_dim]
    conv_out_scale: np.ndarray | None = None    # [conv_dim]
    state_scale: np.ndarray | None = None       # [nh*P] (Mamba1: [d_inner])
    s_y: np.float32 = np.float32(1.0)
    xproj_out_scale: np.ndarray | None = None   # Mamba1 [R+2N]
    s_dt: np.float32 = np.float32(1.0)          # Mamba1 dt_proj output scale
    hadamard: bool = True                       # online H at the out_proj input
    extra: dict = field(default_factory=dict)

    @property
    def A(self):
        return (-np.exp(self.a_log.astype(np.float32))).astype(np.float32)

    @property
    def a8(self):
        return self.profile in ("W8A8", "W4A8")


@dataclass
class QState:
    """Quantized SsmState: int8 h codes + int8 conv-input codes (A8), or f32 (W4A16)."""
    h: np.ndarray              # [nh, P, N] int8 (A8) / f32 (A16)
    conv: np.ndarray           # [conv_dim, K-1] int8 (A8) / f32 (A16)


def zero_qstate(qb: QBlock) -> QState:
    d = qb.dims
    nh, P = (d.n_heads, d.head_dim) if d.variant == "mamba2" else (1, d.d_inner)
    dt = np.int8 if qb.a8 else np.float32
    return QState(np.zeros((nh, P, d.d_state), dt), np.zeros((d.conv_dim, d.conv_kernel - 1), dt))


def _conv_a8(codes, qb: QBlock, cache_codes):
    v = (codes.astype(np.float32) * qb.conv_in_scale[None, :]).astype(np.float32)
    cache = (cache_codes.astype(np.float32) * qb.conv_in_scale[:, None]).astype(np.float32)
    out, _ = causal_conv1d(v, qb.conv_weight, qb.conv_bias, cache)
    K = qb.dims.conv_kernel
    allc = np.concatenate([cache_codes.T, codes], axis=0)
    new_cache = np.ascontiguousarray(allc[allc.shape[0] - (K - 1):].T).astype(np.int8)
    return quantize_codes(out, qb.conv_out_scale[None, :], 8), new_cache


def block_forward_quantized(u, qb: QBlock, state: QState | None = None, chunk=None, trace=None):
    """SPEC.md:326-334 for one sequence u [T×d_model] → (out [T×d_model], QState).
    ``trace`` (dict) receives the intermediate codes for kernel-level parity."""
    d = qb.dims
    st = state if state is not None else zero_qstate(qb)
    u = np.asarray(u, np.float32)
    tr = trace if trace is not None else {}
    if not qb.a8:
        return _block_forward_a16(u, qb, st, tr)
    di = d.d_inner
    uq = quantize_codes(u, qb.s_u, 8)
    y_in, acc_in = qlinear_a8(uq, qb.in_proj, qb.s_u)
    codes = quantize_codes(y_in, qb.in_out_scale[None, :], 8)
    tr.update(u_q=uq, in_acc=acc_in, in_codes=codes)
    z_q = codes[:, :di]
    s_z = qb.in_out_scale[0]
    if d.variant == "mamba2":
        gn = d.n_state_groups * d.d_state
        xbc = codes[:, di:2 * di + 2 * gn]
        dt_q = codes[:, 2 * di + 2 * gn:]
        s_dt = qb.in_out_scale[2 * di + 2 * gn]
        cq, new_conv = _conv_a8(xbc, qb, st.conv)
        tr.update(conv_codes=cq)
        cs = qb.conv_out_scale
        xh = (cq[:, :di].astype(np.float32) * cs[None, :di]).reshape(-1, d.n_heads, d.head_dim)
        Bh = (cq[:, di:di + gn].astype(np.float32) * cs[None, di:di + gn]).reshape(-1, d.n_state_groups, d.d_state)
        Ch = (cq[:, di + gn:].astype(np.float32) * cs[None, di + gn:]).reshape(-1, d.n_state_groups, d.d_state)
        dA, dt = discretize((dt_q.astype(np.float32) * s_dt).astype(np.float32), qb.dt_bias, qb.A)
        zh = (z_q.astype(np.float32) * s_z).astype(np.float32).reshape(-1, d.n_heads, d.head_dim)
        h0 = (st.h.astype(np.float32) * qb.state_scale.reshape(d.n_heads, d.head_dim)[:, :, None]).astype(np.float32)
        y, h = selective_scan(xh, dA, dt, Bh, Ch, qb.d_param, zh, h0, qb.head_group)
        y = y.reshape(-1, di)
        h_q = quantize_codes(h, qb.state_scale.reshape(d.n_heads, d.head_dim)[:, :, None], 8)
    else:
        x_q_in = codes[:, di:2 * di]
        cq, new_conv = _conv_a8(x_q_in, qb, st.conv)
        tr.update(conv_codes=cq)
        yx, _ = qlinear_a8(cq, qb.x_proj, np.float32(1.0))
        xdq = quantize_codes(yx, qb.xproj_out_scale[None, :], 8)
        R, N = d.dt_rank, d.d_state
        s_dtl = qb.xproj_out_scale[0]
        ydt, _ = qlinear_a8(xdq[:, :R], qb.dt_proj, s_dtl)
        dt_q = quantize_codes(ydt, qb.s_dt, 8)
        tr.update(xproj_codes=xdq, dt_codes=dt_q)
        xh = (cq.astype(np.float32) * qb.conv_out_scale[None, :]).astype(np.float32)
        Bm = (xdq[:, R:R + N].astype(np.float32) * qb.xproj_out_scale[R]).astype(np.float32)
        Cm = (xdq[:, R + N:].astype(np.float32) * qb.xproj_out_scale[R + N]).astype(np.float32)
        dA, dt = discretize((dt_q.astype(np.float32) * qb.s_dt).astype(np.float32), qb.dt_bias, qb.A)
        zz = (z_q.astype(np.float32) * s_z).astype(np.float32)
        h0 = (st.h.astype(np.float32).reshape(di, N) * qb.state_scale[:, None]).astype(np.float32)
        y, h = selective_scan(xh, dA, dt, Bm, Cm, qb.d_param, zz, h0)
        h_q = quantize_codes(h.reshape(1, di, N), qb.state_scale.reshape(1, di)[:, :, None], 8)
    tr.update(y=y)
    r = rmsnorm(y, qb.norm_weight, groups=d.norm_groups)
    if qb.hadamard:
        yq = had.hadamard_quantize(r, had.HadamardPlan(di, "none", qb.s_y), 8, d.had_block)
    else:
        yq = quantize_codes(r, qb.s_y, 8)
    out, acc_out = qlinear_a8(yq, qb.out_proj, qb.s_y)
    tr.update(r=r, y_q=yq, out_acc=acc_out, out=out)
    return out, QState(h_q, new_conv)


def _block_forward_a16(u, qb: QBlock, st: QState, tr):
    d = qb.dims
    di = d.d_inner
    zx = qlinear_a16(u, qb.in_proj)
    z = zx[:, :di]
    K = d.conv_kernel
    if d.variant == "mamba2":
        gn = d.n_state_groups * d.d_state
        xbc = zx[:, di:2 * di + 2 * gn]
        dt_raw = zx[:, 2 * di + 2 * gn:]
        conv, cache = causal_conv1d(xbc, qb.conv_weight, qb.conv_bias, st.conv)
        xh = conv[:, :di].reshape(-1, d.n_heads, d.head_dim)
        Bh = conv[:, di:di + gn].reshape(-1, d.n_state_groups, d.d_state)
        Ch = conv[:, di + gn:].reshape(-1, d.n_state_groups, d.d_state)
        dA, dt = discretize(dt_raw, qb.dt_bias, qb.A)
        y, h = selective_scan(xh, dA, dt, Bh, Ch, qb.d_param, z.reshape(-1, d.n_heads, d.head_dim), st.h,
                              qb.head_group)
        y = y.reshape(-1, di)
    else:
        x = zx[:, di:]
        xc, cache = causal_conv1d(x, qb.conv_weight, qb.conv_bias, st.conv)
        R, N = d.dt_rank, d.d_state
        xd = qlinear_a16(xc, qb.x_proj)
        dt_raw = qlinear_a16(xd[:, :R], qb.dt_proj)
        dA, dt = discretize(dt_raw, qb.dt_bias, qb.A)
        y, h = selective_scan(xc, dA, dt, xd[:, R:R + N], xd[:, R + N:], qb.d_param, z,
                              st.h.reshape(di, N))
    r = rmsnorm(y, qb.norm_weight, groups=d.norm_groups)
    out = qlinear_a16(r, qb.out_proj)
    tr.update(in_y=zx, y=y, r=r, out=out)
    return out, QState(np.asarray(h, np.float32).reshape(st.h.shape), cache)


def block_step_batched(u, qb: QBlock, states: list):
    """Decode: one token for each of b independent sequences (rows of u)."""
    outs, new = [], []
    for i in range(u.shape[0]):
        o, s = block_forward_quantized(u[i:i + 1], qb, states[i])
        outs.append(o)
        new.append(s)
    return np.concatenate(outs, axis=0), new


def decode_step_batched(u, qb: QBlock, h_codes, conv_codes, trace=None):
    """Mamba2 A8 decode step for b independent sequences at once (same math as
    ``block_forward_quantized`` with T=1; vectorised over the batch for the CPU
    baseline).  u [b×d_model]; h_codes [b×nh×P×N] int8; conv_codes [b×C×(K-1)] int8.
    Returns (out [b×d_model], h_codes', conv_codes')."""
    d = qb.dims
    di, nh, P, N = d.d_inner, d.n_heads, d.head_dim, d.d_state
    gn = d.n_state_groups * N
    uq = quantize_codes(u, qb.s_u, 8)
    y_in, _ = qlinear_a8(uq, qb.in_proj, qb.s_u)
    codes = quantize_codes(y_in, qb.in_out_scale[None, :], 8)
    xbc = codes[:, di:2 * di + 2 * gn]
    win = np.concatenate([conv_codes, xbc[:, :, None]], axis=2)
    v = (win.astype(np.float32) * qb.conv_in_scale[None, :, None]).astype(np.float32)
    acc = np.broadcast_to(qb.conv_bias[None, :], xbc.shape).astype(np.float32)
    for j in range(d.conv_kernel):
        acc = (acc + (qb.conv_weight[None, :, j] * v[:, :, j]).astype(np.float32)).astype(np.float32)
    from oracle.ssm_block import silu, softplus
    cq = quantize_codes(silu(acc), qb.conv_out_scale[None, :], 8)
    cs = qb.conv_out_scale
    x = (cq[:, :di].astype(np.float32) * cs[None, :di]).reshape(-1, nh, P)
    Bm = (cq[:, di:di + gn].astype(np.float32) * cs[None, di:di + gn]).reshape(-1, d.n_state_groups, N)
    Cm = (cq[:, di + gn:].astype(np.float32) * cs[None, di + gn:]).reshape(-1, d.n_state_groups, N)
    s_dt = qb.in_out_scale[2 * di + 2 * gn]
    dt = softplus((codes[:, 2 * di + 2 * gn:].astype(np.float32) * s_dt).astype(np.float32) + qb.dt_bias[None])
    dA = np.exp((dt * qb.A[None]).astype(np.float32)).astype(np.float32)
    ss = qb.state_scale.reshape(nh, P)[None, :, :, None]
    h = (h_codes.astype(np.float32) * ss).astype(np.float32)
    dtx = (dt[:, :, None] * x).astype(np.float32)
    Bh, Ch = Bm[:, qb.head_group], Cm[:, qb.head_group]
    h = (dA[:, :, None, None] * h + (dtx[..., None] * Bh[:, :, None, :]).astype(np.float32)).astype(np.float32)
    y = (np.einsum("bhpn,bhn->bhp", h.astype(np.float64), Ch.astype(np.float64)).astype(np.float32)
         + (qb.d_param[None, :, None] * x).astype(np.float32))
    z = (codes[:, :di].astype(np.float32) * qb.in_out_scale[0]).reshape(-1, nh, P)
    y = (y * silu(z)).astype(np.float32).reshape(-1, di)
    r = rmsnorm(y, qb.norm_weight, groups=d.norm_groups)
    yq = (had.hadamard_quantize(r, had.HadamardPlan(di, "none", qb.s_y), 8, d.had_block) if qb.hadamard
          else quantize_codes(r, qb.s_y, 8))
    out, _ = qlinear_a8(yq, qb.out_proj, qb.s_y)
    if trace is not None:
        trace.update(in_codes=codes, conv_codes=cq, y=y, y_q=yq)
    return out, quantize_codes(h, ss, 8), np.ascontiguousarray(win[:, :, 1:]).astype(np.int8)
