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
    """A quantized projection.  kind "w8": int8 per-output-channel (s_ch); "w4a8":
    4-bit codes with progressive group scales s_ch·sg (LEDGER G11b); "w4a16": 4-bit
    codes with float group scales s_group (SPEC PerGroup)."""
    kind: str
    codes: np.ndarray
    s_ch: np.ndarray | None = None
    sg: np.ndarray | None = None
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
                self.w = ops.repack_w4(packed, self.N, self.K)
        if self.kind == "w4a8":
            sg = ql.sg
            self.sg = sg if isinstance(sg, torch.Tensor) else _t(np.asarray(sg).astype(np.int8), torch.int8, dev)
        if self.kind == "w4a16":
            sgr = ql.s_group
            self.s_group = sgr if isinstance(sgr, torch.Tensor) else _t(np.asarray(sgr, np.float32), torch.float32, dev)
        else:
            self.s_ch = np.asarray(ql.s_ch, np.float32)
            self.alpha = None
            if s_a is not None:
                self.set_input_scale(s_a)

    def set_input_scale(self, s_a: float):
        """alpha[n] = f32(s_ch[n] · s_a) (fuse_scales)."""
        dev = self.w.device
        self.alpha = _t((self.s_ch * np.float32(s_a)).astype(np.float32), torch.float32, dev)

    def a8(self, a_codes, epi, out=None, col_scale=None, gsum=None):
        """``gsum``: optional int32 128-block sums of ``a_codes`` (W4A8 offset correction)."""
        if self.kind == "w8":
            return ops.gemm_w8a8(a_codes, self.w, self.alpha, epi, out, col_scale)
        if self.kind == "w4a8":
            return ops.gemm_w4a8(a_codes, self.w, self.sg, self.group, self.alpha, self.N, epi, out, col_scale, gsum)
        raise ShapeError("A8 GEMM on a W4A16 projection")

    def a16(self, x, out=None, resid=False):
        return ops.gemv_w4a16(x, self.w, self.s_group, self.group, self.N, out, resid)

    @property
    def nbytes(self):
        n = self.w.numel() * self.w.element_size()
        if self.kind == "w4a8":
            n += self.sg.numel()
        if self.kind == "w4a16":
            n += self.s_group.numel() * 4
        else:
            n += self.N * 4
        return n


class DeviceBlock:
    """One quantized block resident on the GPU (weights, scale tables, kernel params)."""

    def __init__(self, qb, dev="cuda"):
        d = qb.dims
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
    def forward_codes(self, u_codes, B, T, state: SsmState, state_in: bool, resid=None, ws=None, u_gsum=None):
        """A8 block on int8 input codes [B*T × d_model].  If ``resid`` is given the out_proj
        epilogue adds into it (residual stream) and it is returned; else returns f32 out."""
        d = self.dims
        di = d.d_inner
        M = B * T
        ws = ws if ws is not None else {}
        zx = self.in_proj.a8(u_codes, ops.EPI_QUANT, ws.get("zx"), self.in_out_scale, u_gsum)
        y = ws.get("y")
        if y is None:
            y = torch.empty((M, di), dtype=torch.float32, device=u_codes.device)
        if d.variant == "mamba2":
            gn = d.n_state_groups * d.d_state
            xbc = zx[:, di:2 * di + 2 * gn]
            if T == 1 and state_in and self.fused_decode:
                # conv update + int8 state update + gated norm + FWHT + quant (sq_mamba2_decode_step_int8)
                ygs = ws.get("yq_gs") if self.profile == "W4A8" else None   # block sums feed W4A8 only
                yq = ops.mamba2_decode_step_int8(self.decode_params, B, zx, state.conv_cache, state.h, ws.get("yq"),
                                                 y, ws.get("dws"), ygs)
                if resid is not None:
                    return self.out_proj.a8(yq, ops.EPI_RESID, resid, gsum=ygs)
                return self.out_proj.a8(yq, ops.EPI_F32, ws.get("out"), gsum=ygs)
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

    def forward_a16(self, u, B, T, state: SsmState, state_in: bool, resid=None, ws=None):
        """W4A16 float path on f32 input u [B*T × d_model]."""
        d = self.dims
        di = d.d_inner
        ws = ws if ws is not None else {}
        zx = self.in_proj.a16(u, ws.get("zxf"))
        if d.variant == "mamba1":   # in_proj rows z | x; x_proj rows Δ_low | B | C (LEDGER G4)
            R = d.dt_rank
            cv = ops.conv1d_f32(zx[:, di:], self.conv_w, self.conv_b, B, T, state.conv_cache, state_in,
                                ws.get("convf"))
            xd = self.x_proj.a16(cv)
            dtr = self.dt_proj.a16(xd[:, :R])
            y = ws.get("y")
            if y is None:
                y = torch.empty((B * T, di), dtype=torch.float32, device=u.device)
            ops.selective_scan_f32(self.params, B, T, cv, dtr, xd[:, R:], zx[:, :di], state.h, state_in, y)
            r = ops.rmsnorm_f32(y, self.norm_w, EPS_NORM, ws.get("r"))
            if resid is not None:
                return self.out_proj.a16(r, resid, resid=True)
            return self.out_proj.a16(r, ws.get("out"))
        gn = d.n_state_groups * d.d_state
        xbc = zx[:, di:2 * di + 2 * gn]
        cv = ops.conv1d_f32(xbc, self.conv_w, self.conv_b, B, T, state.conv_cache, state_in, ws.get("convf"))
        y = ws.get("y")
        if y is None:
            y = torch.empty((B * T, di), dtype=torch.float32, device=u.device)
        ops.ssd_scan_f32(self.params, B, T, cv[:, :di], cv[:, di:di + gn], cv[:, di + gn:], zx[:, 2 * di + 2 * gn:],
                         zx[:, :di], state.h, state_in, y)
        r = ops.rmsnorm_f32(y, self.norm_w, EPS_NORM, ws.get("r"))
        if resid is not None:
            return self.out_proj.a16(r, resid, resid=True)
        return self.out_proj.a16(r, ws.get("out"))


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
