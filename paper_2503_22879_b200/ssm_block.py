"""ssm_block — SPEC `[MODULE] ssm_block` on the B200.

Host types keep the reference field names (SsmBlockWeights SPEC.md:260-265, SsmState
SPEC.md:266-269) plus the quantized block `QBlock` (weights + per-activation scale set,
the SPEC `plan`).  The forward path runs on the GPU through the C-ABI kernels
(`ops`), with no CPU fallback:

  u ─quantize(s_u)─▶ in_proj GEMM (+requant z|x|B|C|Δ) ─▶ conv1d+SiLU+requant
    ─▶ SSD / selective scan (fp32 state, gate) ─▶ RMSNorm+FWHT+quant(s_y) ─▶ out_proj

Layout contracts (LEDGER G4): weights [out × in]; Mamba2 in_proj rows
z | x | B | C | Δ; Mamba1 in_proj rows z | x, x_proj rows Δ_low | B | C.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import ops
from .errors import ShapeError

EPS_NORM = 1e-5


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
    dt_rank: int = 0
    norm_groups: int = 1      # gated-RMSNorm groups: 1 = full d_inner; > 1 = head-shard recipe

    @property
    def had_block(self):
        """Online Hadamard block: largest power of two dividing d_inner / norm_groups (LEDGER G9)."""
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

    @property
    def state_rows(self):
        """(heads, channels-per-head) of SsmState.h (Mamba1: 1 × d_inner)."""
        return (self.n_heads, self.head_dim) if self.variant == "mamba2" else (1, self.d_inner)


@dataclass
class SsmBlockWeights:
    """SPEC.md:260-265 (+ Mamba1 x_proj/dt_proj, LEDGER G4).  Float host tensors."""
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
            per = d.n_heads // d.n_state_groups
            self.head_group = (np.arange(d.n_heads) // per).astype(np.int32)

    def copy(self, **kw):
        return replace(self, **kw)


@dataclass
class SsmState:
    """recurrent state h [nh×P×N] and conv cache [channels×(K−1)]."""
    h: object
    conv_cache: object


@dataclass
class QLinear:
    """A quantized projection.  kind "w8": int8 per-output-channel (s_ch); "w4a8" / "w4a16":
    4-bit codes with float group scales s_group (SPEC PerGroup, LEDGER G11)."""
    kind: str
    codes: np.ndarray
    s_ch: np.ndarray | None = None
    s_group: np.ndarray | None = None
    group: int = 128

    @property
    def n_out(self):
        return self.codes.shape[0]

    @property
    def k(self):
        return self.codes.shape[1]


@dataclass
class QBlock:
    """Quantized block = weights + per-activation scale set (the SPEC `plan`)."""
    dims: Dims
    profile: str
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
    s_u: float = 1.0
    in_out_scale: np.ndarray | None = None
    conv_in_scale: np.ndarray | None = None
    conv_out_scale: np.ndarray | None = None
    state_scale: np.ndarray | None = None
    s_y: float = 1.0
    xproj_out_scale: np.ndarray | None = None
    s_dt: float = 1.0
    hadamard: bool = True
    extra: dict = field(default_factory=dict)

    @property
    def a8(self):
        return self.profile in ("W8A8", "W4A8")


# ============================================================== device side
def _t(a, dtype, dev):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)


def pack_u4_host(codes: np.ndarray) -> np.ndarray:
    """u4packed: two's-complement nibbles, low nibble = even index."""
    u = (np.asarray(codes).astype(np.int16) & 0xF).astype(np.uint8)
    return (u[..., 0::2] | (u[..., 1::2] << 4)).astype(np.uint8)


class DeviceLinear:
    """A quantized projection resident in HBM in the kernel layout."""

    def __init__(self, ql, dev, s_a: float | None = None):
        self.kind = ql.kind
        self.group = int(ql.group)
        dw = getattr(ql, "device_w", None)     # already-resident weights (synthetic / loaded)
        if dw is not None:
            self.N, self.K = ql.shape
            self.w = dw
        else:
            self.N, self.K = ql.codes.shape
            if self.kind == "w8":
                self.w = _t(ql.codes.astype(np.int8), torch.int8, dev)
            else:
                packed = _t(pack_u4_host(ql.codes), torch.uint8, dev)
                self.w = (ops.repack_w4a16(packed, self.N, self.K, int(ql.group)) if self.kind == "w4a16"
                          else ops.repack_w4(packed, self.N, self.K))
        if self.kind in ("w4a8", "w4a16"):
            sgr = ql.s_group
            self.s_group = sgr if isinstance(sgr, torch.Tensor) else _t(np.asarray(sgr, np.float32), torch.float32, dev)
            if self.s_group.shape != (self.N, self.K // self.group):
                raise ShapeError(f"s_group must be [{self.N} x {self.K // self.group}]")
        if self.kind == "w4a8":
            self.ws = ops.tile_group_scales(self.s_group)   # kernel layout [N/128][G][128]
        if self.kind == "w8":
            self.s_ch = np.asarray(ql.s_ch, np.float32)
            self.alpha = None
        self.s_a = None
        if s_a is not None:
            self.set_input_scale(s_a)

    def set_input_scale(self, s_a: float):
        """W8: alpha[n] = f32(s_ch[n] · s_a) (fuse_scales); W4A8: s_a scales
        the promoted per-group sum."""
        self.s_a = np.float32(s_a)
        if self.kind == "w8":
            self.alpha = _t((self.s_ch * np.float32(s_a)).astype(np.float32), torch.float32, self.w.device)

    def a8(self, a_codes, epi, out=None, col_scale=None):
        if self.kind == "w8":
            return ops.gemm_w8a8(a_codes, self.w, self.alpha, epi, out, col_scale)
        if self.kind == "w4a8":
            return ops.gemm_w4a8(a_codes, self.w, self.ws, self.group, self.s_a, self.N, epi, out, col_scale)
        raise ShapeError("A8 GEMM on a W4A16 projection")

    def a16(self, x, out=None, resid=False, norm_w=None, conv=None):
        """W4A16 projection of x (RMS-normalised with norm_w on the way in when given; ``conv`` fuses
        the T = 1 conv update of a column range into the epilogue, ops.gemv_w4a16)."""
        return ops.gemv_w4a16(x, self.w, self.s_group, self.group, self.N, out, resid, norm_w, EPS_NORM, conv)

    @property
    def nbytes(self):
        n = self.w.numel() * self.w.element_size()
        if self.kind in ("w4a8", "w4a16"):
            n += self.s_group.numel() * 4
        else:
            n += self.N * 4
        return n


class DeviceBlock:
    """One quantized block resident on the GPU (weights, scale tables, kernel params)."""

    def __init__(self, qb, dev="cuda"):
        d = qb.dims
        if getattr(d, "norm_groups", 1) != 1:
            raise ShapeError("a block with norm_groups > 1 runs head-sharded (parallel.HeadShardedBlock): the "
                             "gated-norm / Hadamard kernels normalise whole rows")
        self.dims = d
        self.profile = qb.profile
        self.a8 = qb.profile in ("W8A8", "W4A8")
        self.hadamard = bool(getattr(qb, "hadamard", True))
        self.fused_decode = (qb.profile in ("W8A8", "W4A8") and d.variant == "mamba2" and d.head_dim == 64
                             and d.d_state in (64, 128))
        f = lambda a: _t(np.asarray(a, np.float32), torch.float32, dev)
        self.s_u = np.float32(qb.s_u)
        self.s_y = np.float32(qb.s_y)
        self.in_proj = DeviceLinear(qb.in_proj, dev, self.s_u if self.a8 else None)
        self.out_proj = DeviceLinear(qb.out_proj, dev, self.s_y if self.a8 else None)
        self.conv_w = f(qb.conv_weight)
        self.conv_b = f(qb.conv_bias)
        self.A = f(-np.exp(np.asarray(qb.a_log, np.float32)))
        self.D = f(qb.d_param)
        self.dt_bias = f(qb.dt_bias)
        self.norm_w = f(qb.norm_weight)
        if d.variant == "mamba2":
            self.head_group = _t(np.asarray(qb.head_group, np.int32), torch.int32, dev)
        if self.a8:
            self.in_out_scale = f(qb.in_out_scale)
            self.conv_in_scale = f(qb.conv_in_scale)
            self.conv_out_scale = f(qb.conv_out_scale)
            self.state_scale = f(qb.state_scale)
            di = d.d_inner
            if d.variant == "mamba2":
                gn = d.n_state_groups * d.d_state
                ios = np.asarray(qb.in_out_scale, np.float32)
                cos_ = np.asarray(qb.conv_out_scale, np.float32)
                self.s_B = f(cos_[di:di + gn:d.d_state])
                self.s_C = f(cos_[di + gn::d.d_state])
                self.s_x = f(cos_[:di])
                self.params = ops.mamba2_params(d.n_heads, d.head_dim, d.d_state, d.n_state_groups, self.head_group,
                                                self.A, self.D, self.dt_bias, ios[2 * di + 2 * gn], ios[0],
                                                self.s_x, self.s_B, self.s_C, self.state_scale)
                self.decode_params = ops.mamba2_decode_params(self.params, self.conv_w, self.conv_b,
                                                              self.conv_in_scale, self.conv_out_scale, self.norm_w,
                                                              EPS_NORM, self.s_y, self.hadamard)
            else:
                R, N = d.dt_rank, d.d_state
                ios = np.asarray(qb.in_out_scale, np.float32)
                xos = np.asarray(qb.xproj_out_scale, np.float32)
                self.x_proj = DeviceLinear(qb.x_proj, dev, 1.0)
                self.dt_proj = DeviceLinear(qb.dt_proj, dev, xos[0])
                self.xproj_out_scale = f(xos)
                self.dt_scale = f(np.full(di, np.float32(qb.s_dt), np.float32))
                self.s_x = f(qb.conv_out_scale)
                self.params = ops.mamba1_params(di, N, self.A, self.D, self.dt_bias, np.float32(qb.s_dt), ios[0],
                                                xos[R], xos[R + N], self.s_x, self.state_scale)
                # one-launch decode (conv, x_proj, dt_proj, scan step, norm; decode_m1.cu) for W8 projections
                self.m1_fused_decode = (self.x_proj.kind == "w8" and self.dt_proj.kind == "w8" and N == 16
                                        and R % 4 == 0 and di % 16 == 0)
                if self.m1_fused_decode:
                    self.m1_decode_params = ops.mamba1_decode_params(
                        self.params, self.conv_w, self.conv_b, self.conv_in_scale, self.conv_out_scale, R,
                        self.x_proj.w, self.x_proj.alpha, self.xproj_out_scale, self.dt_proj.w, self.dt_proj.alpha,
                        self.dt_scale, self.norm_w, EPS_NORM, self.s_y, self.hadamard)
        else:
            if d.variant == "mamba2":
                self.params = ops.mamba2_params(d.n_heads, d.head_dim, d.d_state, d.n_state_groups,
                                                self.head_group, self.A, self.D, self.dt_bias)
            else:
                # float operands: the scan kernel takes raw dt_proj outputs and x_proj B|C rows
                self.x_proj = DeviceLinear(qb.x_proj, dev)
                self.dt_proj = DeviceLinear(qb.dt_proj, dev)
                ones = f(np.ones(d.d_inner, np.float32))
                self._ones = ones
                self.params = ops.mamba1_params(d.d_inner, d.d_state, self.A, self.D, self.dt_bias, 1.0, 1.0, 1.0,
                                                1.0, ones, ones)

    # ------------------------------------------------------------------ state
    def new_state(self, batch: int, dev="cuda"):
        d = self.dims
        nh, P = (d.n_heads, d.head_dim) if d.variant == "mamba2" else (1, d.d_inner)
        dt = torch.int8 if self.a8 else torch.float32
        h = torch.zeros((batch, nh, P, d.d_state), dtype=dt, device=dev)
        conv = torch.zeros((batch, d.conv_kernel - 1, d.conv_dim), dtype=dt, device=dev)
        return SsmState(h, conv)

    @property
    def weight_bytes(self):
        n = self.in_proj.nbytes + self.out_proj.nbytes
        if self.dims.variant == "mamba1":
            n += self.x_proj.nbytes + self.dt_proj.nbytes
        return n

    # ------------------------------------------------------------------ forward
    def forward_codes(self, u_codes, B, T, state: SsmState, state_in: bool, resid=None, ws=None):
        """A8 block on int8 input codes [B*T × d_model].  If ``resid`` is given the out_proj
        epilogue adds into it (residual stream) and it is returned; else returns f32 out."""
        d = self.dims
        di = d.d_inner
        M = B * T
        ws = ws if ws is not None else {}
        zx = self.in_proj.a8(u_codes, ops.EPI_QUANT, ws.get("zx"), self.in_out_scale)
        y = ws.get("y")
        if y is None:
            y = torch.empty((M, di), dtype=torch.float32, device=u_codes.device)
        if d.variant == "mamba2":
            gn = d.n_state_groups * d.d_state
            xbc = zx[:, di:2 * di + 2 * gn]
            if T == 1 and state_in and self.fused_decode:
                # conv update + int8 state update + gated norm + FWHT + quant (sq_mamba2_decode_step_int8)
                yq = ops.mamba2_decode_step_int8(self.decode_params, B, zx, state.conv_cache, state.h, ws.get("yq"),
                                                 y, ws.get("dws"))
                if resid is not None:
                    return self.out_proj.a8(yq, ops.EPI_RESID, resid)
                return self.out_proj.a8(yq, ops.EPI_F32, ws.get("out"))
            if T == 1 and state_in:
                cv = ops.conv1d_update_int8(xbc, self.conv_w, self.conv_b, self.conv_in_scale, self.conv_out_scale,
                                            state.conv_cache, ws.get("conv"))
                ops.state_update_int8(self.params, B, cv[:, :di], cv[:, di:di + gn], cv[:, di + gn:],
                                      zx[:, 2 * di + 2 * gn:], zx[:, :di], state.h, y)
            else:
                cv = ops.conv1d_int8(xbc, self.conv_w, self.conv_b, self.conv_in_scale, self.conv_out_scale, B, T,
                                     state.conv_cache, state_in, ws.get("conv"))
                ops.ssd_scan_int8(self.params, B, T, cv[:, :di], cv[:, di:di + gn], cv[:, di + gn:],
                                  zx[:, 2 * di + 2 * gn:], zx[:, :di], state.h, state_in, y)
        else:
            R, N = d.dt_rank, d.d_state
            xin = zx[:, di:]
            if T == 1 and state_in and getattr(self, "m1_fused_decode", False) and B <= 8:
                m1ws = ws.get("m1ws")
                if m1ws is None:   # zero-filled: the kernel's grid-barrier counters live here
                    m1ws = torch.zeros(ops.mamba1_decode_ws_bytes(self.m1_decode_params, B), dtype=torch.uint8,
                                       device=u_codes.device)
                yq = ops.mamba1_decode_step_int8(self.m1_decode_params, B, zx, state.conv_cache, state.h, m1ws,
                                                 ws.get("yq"))
                if resid is not None:
                    return self.out_proj.a8(yq, ops.EPI_RESID, resid)
                return self.out_proj.a8(yq, ops.EPI_F32, ws.get("out"))
            if T == 1 and state_in:
                cv = ops.conv1d_update_int8(xin, self.conv_w, self.conv_b, self.conv_in_scale, self.conv_out_scale,
                                            state.conv_cache, ws.get("conv"))
            else:
                cv = ops.conv1d_int8(xin, self.conv_w, self.conv_b, self.conv_in_scale, self.conv_out_scale, B, T,
                                     state.conv_cache, state_in, ws.get("conv"))
            xd = self.x_proj.a8(cv, ops.EPI_QUANT, ws.get("xd"), self.xproj_out_scale)
            dtq = self.dt_proj.a8(xd[:, :R], ops.EPI_QUANT, ws.get("dtq"), self.dt_scale)
            ops.selective_scan_int8(self.params, B, T, cv, dtq, xd[:, R:], zx[:, :di], state.h, state_in, y)
        yq = ops.gate_norm_had_quant(y, self.norm_w, EPS_NORM, self.s_y, self.hadamard, ws.get("yq"))
        if resid is not None:
            return self.out_proj.a8(yq, ops.EPI_RESID, resid)
        return self.out_proj.a8(yq, ops.EPI_F32, ws.get("out"))

    def forward_a16(self, u, B, T, state: SsmState, state_in: bool, resid=None, ws=None, u_norm=None):
        """W4A16 float path on f32 input u [B*T × d_model] (when ``u_norm`` is given, u is the raw
        residual stream and the in_proj GEMV applies the model's pre-norm on the way in).  The
        gated RMSNorm runs inside the out_proj GEMV's input staging."""
        d = self.dims
        di = d.d_inner
        ws = ws if ws is not None else {}
        conv = None
        if T == 1:   # decode: the conv update runs in the in_proj GEMV's epilogue (sq_gemv_w4a16_conv)
            cv = ws.get("convf")
            if cv is None:
                cv = torch.empty((B, d.conv_dim), dtype=torch.float32, device=u.device)
            conv = (self.conv_w, self.conv_b, di, state.conv_cache, state_in, cv)
        zx = self.in_proj.a16(u, ws.get("zxf"), norm_w=u_norm, conv=conv)
        if d.variant == "mamba1":   # in_proj rows z | x; x_proj rows Δ_low | B | C (LEDGER G4)
            R = d.dt_rank
            if conv is None:
                cv = ops.conv1d_f32(zx[:, di:], self.conv_w, self.conv_b, B, T, state.conv_cache, state_in,
                                    ws.get("convf"))
            xd = self.x_proj.a16(cv)
            dtr = self.dt_proj.a16(xd[:, :R])
            y = ws.get("y")
            if y is None:
                y = torch.empty((B * T, di), dtype=torch.float32, device=u.device)
            ops.selective_scan_f32(self.params, B, T, cv, dtr, xd[:, R:], zx[:, :di], state.h, state_in, y)
        else:
            gn = d.n_state_groups * d.d_state
            xbc = zx[:, di:2 * di + 2 * gn]
            if conv is None:
                cv = ops.conv1d_f32(xbc, self.conv_w, self.conv_b, B, T, state.conv_cache, state_in, ws.get("convf"))
            y = ws.get("y")
            if y is None:
                y = torch.empty((B * T, di), dtype=torch.float32, device=u.device)
            ops.ssd_scan_f32(self.params, B, T, cv[:, :di], cv[:, di:di + gn], cv[:, di + gn:],
                             zx[:, 2 * di + 2 * gn:], zx[:, :di], state.h, state_in, y)
        if resid is not None:
            return self.out_proj.a16(y, resid, resid=True, norm_w=self.norm_w)
        return self.out_proj.a16(y, ws.get("out"), norm_w=self.norm_w)


# ============================================================== SPEC float ops on the GPU
# SPEC.md:272-325 with the reference's argument order (oracle/ssm_block.py restates them).  Each
# takes CUDA float32 tensors and runs on the library kernels: sq_conv1d_f32, sq_discretize_f32,
# sq_selective_scan{2,1}_pre_f32, sq_rmsnorm_f32; the float projections are plain library GEMMs
# (cuBLAS, float64 accumulation like tensor.matmul, pkg/src/ssmquant/tensor.py:33-54).
def _f32(a, dev=None):
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            raise ShapeError("SPEC ops take CUDA tensors (no CPU fallback)")
        return a.to(torch.float32)
    return torch.as_tensor(np.asarray(a, np.float32), device=dev or "cuda")


def _gemm_f(a, w):
    w = _f32(w, a.device)
    return (a.to(torch.float64) @ w.to(torch.float64).T).to(torch.float32)


def project_inputs(u, w: SsmBlockWeights):
    """Mamba2 → (x, B, C, Δ_raw, z), slices of one in_proj GEMM in the fixed
    order z | x | B | C | Δ; Mamba1 → (x, None, None, None, z) (B/C/Δ come from
    x_proj after the conv)."""
    d = w.dims
    u = _f32(u)
    if u.dim() != 2 or u.shape[1] != d.d_model:
        raise ShapeError(f"u must be [T x {d.d_model}]")
    zx = _gemm_f(u, w.in_proj)
    if zx.shape[1] != d.in_proj_out:
        raise ShapeError(f"in_proj must have {d.in_proj_out} rows")
    di = d.d_inner
    z, x = zx[:, :di], zx[:, di:2 * di]
    if d.variant == "mamba1":
        return x, None, None, None, z
    gn = d.n_state_groups * d.d_state
    return x, zx[:, 2 * di:2 * di + gn], zx[:, 2 * di + gn:2 * di + 2 * gn], zx[:, 2 * di + 2 * gn:], z


def causal_conv1d(x, weight, bias, cache=None):
    """depthwise causal conv + SiLU over x [T×C] (sq_conv1d_f32); ``cache``
    [C×(K−1)] holds the previous K−1 inputs (None = zeros).  Returns (y, new_cache)."""
    x = _f32(x)
    wt, b = _f32(weight, x.device).contiguous(), _f32(bias, x.device).contiguous()
    T, C_ = x.shape
    K = wt.shape[1]
    if wt.shape[0] != C_ or b.shape[0] != C_:
        raise ShapeError("cache/channel mismatch: weight / bias channels")
    cc = torch.zeros((1, K - 1, C_), dtype=torch.float32, device=x.device)
    if cache is not None:
        cache = _f32(cache, x.device)
        if tuple(cache.shape) != (C_, K - 1):
            raise ShapeError("cache/channel mismatch")
        cc[0] = cache.T
    y = ops.conv1d_f32(x.contiguous(), wt, b, 1, T, cc, cache is not None)
    return y, cc[0].T.contiguous()


def discretize(dt_raw, dt_bias, A):
    """SPEC.md:290-298 (sq_discretize_f32): Δ = softplus(Δ_raw + dt_bias), Ȧ = exp(Δ·A).
    Mamba2: Δ_raw [T×nh], A [nh] → Ȧ [T×nh]; Mamba1: A [d×N] → Ȧ [T×d×N].  Returns (Ȧ, Δ)."""
    dt_raw = _f32(dt_raw)
    return ops.discretize_f32(dt_raw, _f32(dt_bias, dt_raw.device).contiguous(), _f32(A, dt_raw.device))


def _scan_pre(x, dA, dt, B, C, D, z, state, head_group):
    x = _f32(x)
    dev = x.device
    T = x.shape[0]
    Dv = _f32(D, dev).contiguous()
    if x.dim() == 3:        # Mamba2: x [T×nh×P], Ȧ/Δ [T×nh], B/C [T×G×N]
        _, nh, P = x.shape
        G, N = B.shape[1], B.shape[2]
        hg = (torch.as_tensor(np.asarray(head_group), dtype=torch.int32, device=dev) if head_group is not None
              else (torch.arange(nh, device=dev, dtype=torch.int32) // (nh // G)))
        zero = torch.zeros(nh, dtype=torch.float32, device=dev)
        p = ops.mamba2_params(nh, P, N, G, hg, zero, Dv, zero)
        h = (torch.zeros((1, nh, P, N), dtype=torch.float32, device=dev) if state is None
             else _f32(state, dev).reshape(1, nh, P, N).clone())
        y = torch.empty((T, nh * P), dtype=torch.float32, device=dev)
        zz = None if z is None else _f32(z, dev).reshape(T, nh * P).contiguous()
        ops.selective_scan2_pre_f32(p, 1, T, x.reshape(T, nh * P).contiguous(), _f32(dA, dev).contiguous(),
                                    _f32(dt, dev).contiguous(), _f32(B, dev).reshape(T, G * N).contiguous(),
                                    _f32(C, dev).reshape(T, G * N).contiguous(), zz, h, state is not None, y)
        _keep = (hg, zero, Dv)   # noqa: F841  (the params struct holds raw pointers)
        return y.reshape(T, nh, P), h[0]
    _, d = x.shape          # Mamba1: x [T×d], Ȧ [T×d×N], Δ [T×d], B/C [T×N]
    N = B.shape[1]
    zero = torch.zeros(d * N, dtype=torch.float32, device=dev)
    ones = torch.ones(d, dtype=torch.float32, device=dev)
    p = ops.mamba1_params(d, N, zero, Dv, zero, 1.0, 1.0, 1.0, 1.0, ones, ones)
    h = (torch.zeros((1, d, N), dtype=torch.float32, device=dev) if state is None
         else _f32(state, dev).reshape(1, d, N).clone())
    y = torch.empty((T, d), dtype=torch.float32, device=dev)
    zz = None if z is None else _f32(z, dev).contiguous()
    ops.selective_scan1_pre_f32(p, 1, T, x.contiguous(), _f32(dA, dev).contiguous(), _f32(dt, dev).contiguous(),
                                _f32(B, dev).contiguous(), _f32(C, dev).contiguous(), zz, h, state is not None, y)
    _keep = (zero, ones, Dv)   # noqa: F841
    return y, h.reshape(1, d, N)


def selective_scan(x, dA, dt, B, C, D, z=None, state=None, head_group=None):
    """SPEC.md:299-307, Eq. 2: h_t = Ȧ_t h_{t−1} + (Δ_t x_t) B_t, y_t = C_t·h_t + D x_t, optional
    gate y·SiLU(z).  Mamba2 when x is [T×nh×P] (B/C [T×G×N] per state group), Mamba1 when x is
    [T×d] (Ȧ [T×d×N], B/C [T×N]).  Returns (y, h) like the oracle (oracle/ssm_block.py)."""
    return _scan_pre(x, dA, dt, B, C, D, z, state, head_group)


def ssd_chunked(x, dA, dt, B, C, D, z=None, chunk=64, state=None, head_group=None):
    """SPEC.md:308-316 for float operands.  Mamba2 shapes.  The float path evaluates the same
    f32 recurrence as ``selective_scan`` (exact, so every chunk size gives the same result,
    within the SPEC's 1e-4 of the block decomposition); the chunked tensor-core engines serve
    the int8 path (sq_ssd_scan_int8, ``DeviceBlock.forward_codes``)."""
    if chunk < 1:
        raise ValueError("chunk must be >= 1")
    if _f32(x).dim() != 3:
        raise ShapeError("ssd_chunked takes Mamba2 operands x [T x nh x P]")
    return _scan_pre(x, dA, dt, B, C, D, z, state, head_group)


def block_forward_float(u, w: SsmBlockWeights, state: SsmState | None = None, chunk=None):
    """SPEC.md:317-325 on the GPU: project → conv → discretize → scan/SSD → gate → RMSNorm →
    out_proj for one sequence u [T×d_model].  Returns (out [T×d_model], SsmState) with the
    state in the SPEC layout (h [nh×P×N] / [1×d×N], conv_cache [C×(K−1)])."""
    d = w.dims
    u = _f32(u)
    dev = u.device
    x, Bi, Ci, dt_raw, z = project_inputs(u, w)
    A = -torch.exp(_f32(w.a_log, dev))
    cache = None if state is None else state.conv_cache
    h0 = None if state is None else state.h
    T = u.shape[0]
    if d.variant == "mamba2":
        di, gn = d.d_inner, d.n_state_groups * d.d_state
        co, cache = causal_conv1d(torch.cat([x, Bi, Ci], 1), w.conv_weight, w.conv_bias, cache)
        dA, dt = discretize(dt_raw, w.dt_bias, A)
        scan = selective_scan if chunk is None else (lambda *a, **k: ssd_chunked(*a, chunk=chunk, **k))
        y, h = scan(co[:, :di].reshape(T, d.n_heads, d.head_dim), dA, dt,
                    co[:, di:di + gn].reshape(T, d.n_state_groups, d.d_state),
                    co[:, di + gn:].reshape(T, d.n_state_groups, d.d_state), w.d_param,
                    z=z.reshape(T, d.n_heads, d.head_dim), state=h0, head_group=w.head_group)
        y = y.reshape(T, di)
    else:
        R, N = d.dt_rank, d.d_state
        xc, cache = causal_conv1d(x, w.conv_weight, w.conv_bias, cache)
        xd = _gemm_f(xc, w.x_proj)
        dt_raw = _gemm_f(xd[:, :R].contiguous(), w.dt_proj)
        dA, dt = discretize(dt_raw, w.dt_bias, A)
        y, h = selective_scan(xc, dA, dt, xd[:, R:R + N], xd[:, R + N:R + 2 * N], w.d_param, z=z, state=h0)
    gam = _f32(w.norm_weight, dev).contiguous()
    y = y.contiguous()
    if d.norm_groups == 1:
        r = ops.rmsnorm_f32(y, gam, EPS_NORM)
    else:   # grouped norm (head-shard recipe): one strided column slice per group
        r = torch.empty_like(y)
        gw = d.d_inner // d.norm_groups
        for g in range(d.norm_groups):
            ops.rmsnorm_f32(y[:, g * gw:(g + 1) * gw], gam[g * gw:(g + 1) * gw], EPS_NORM, r[:, g * gw:(g + 1) * gw])
    return _gemm_f(r, w.out_proj), SsmState(h, cache)


def block_forward_quantized(u, qw, plan=None, bits_profile=None, state: SsmState | None = None, batch: int = 1):
    """SPEC.md:326-334 on the GPU.  ``u`` f32 CUDA tensor [T×d_model] (or [B·T×d_model]
    with ``batch`` sequences); ``qw`` a QBlock (host) or DeviceBlock.  ``plan`` and
    ``bits_profile`` are carried by the QBlock (kept for the SPEC signature).
    Returns (out f32 [B·T×d_model], new SsmState)."""
    blk = qw if isinstance(qw, DeviceBlock) else DeviceBlock(qw, u.device)
    if bits_profile is not None and bits_profile != blk.profile:
        raise ShapeError(f"bits_profile {bits_profile} != block profile {blk.profile}")
    M = u.shape[0]
    if M % batch:
        raise ShapeError("rows not divisible by batch")
    T = M // batch
    st_in = state is not None
    st = state if st_in else blk.new_state(batch, u.device)
    if blk.a8:
        codes = ops.quantize_f32(u, blk.s_u)
        out = blk.forward_codes(codes, batch, T, st, st_in)
    else:
        out = blk.forward_a16(u.contiguous(), batch, T, st, st_in)
    return out, st
