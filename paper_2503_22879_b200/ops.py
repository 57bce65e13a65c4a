"""Torch-tensor wrappers over the C-ABI (one function per `sq_*` entry point).

Every wrapper validates device/dtype/layout, passes raw device pointers plus the current
torch stream, and maps a non-zero status to the ``errors`` hierarchy.  There is no CPU
path: a tensor that is not on a CUDA device raises ``LayoutError``.
2-D operands may be row-strided views (``t[:, a:b]``); their last dim must be dense.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .errors import LayoutError, ShapeError, status_error

EPI_I32, EPI_F32, EPI_QUANT, EPI_RESID = 0, 1, 2, 3


def lib():
    return _lib.load()


LAUNCH_COUNTER = [0, 0]   # [kernel launches issued through this module, launches in last captured step]


def _check(rc: int, launches: int = 1):
    """Map a C-ABI status onto the errors hierarchy; ``launches`` = kernels the call issued."""
    LAUNCH_COUNTER[0] += launches
    if rc != 0:
        raise status_error(rc, _lib.last_error())


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _need(t: torch.Tensor, n: int, name: str):
    """Buffers the kernels index by the launch dimensions must hold at least n elements."""
    if t.numel() < n:
        raise ShapeError(f"{name} must hold at least {n} elements, got {t.numel()}")


def _rows(t: torch.Tensor, n: int, name: str):
    if t.dim() >= 1 and t.shape[0] < n:
        raise ShapeError(f"{name} must have at least {n} rows, got {t.shape[0]}")


def _dev(t: torch.Tensor, dtype, name, dims=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise LayoutError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise LayoutError(f"{name} must be {dtype}, got {t.dtype}")
    if dims is not None and t.dim() != dims:
        raise ShapeError(f"{name} must be {dims}-D, got {tuple(t.shape)}")
    if t.dim() >= 1 and t.numel() > 0 and t.stride(-1) != 1:
        raise LayoutError(f"{name} last dim must be contiguous")
    if t.dim() > 2 and not t.is_contiguous():
        raise LayoutError(f"{name} must be contiguous")
    return t.data_ptr()


def _ld(t):
    return t.stride(0) if t.dim() >= 2 else t.shape[-1]


def _opt(t):
    return 0 if t is None else t.data_ptr()


# ------------------------------------------------------------------ weights
def w4_bytes(N: int, K: int) -> int:
    return int(lib().sq_w4_bytes(N, K))


def repack_w4(u4packed: torch.Tensor, N: int, K: int) -> torch.Tensor:
    _dev(u4packed, torch.uint8, "u4packed")
    if u4packed.numel() != N * K // 2:
        raise ShapeError("u4packed must hold N*K/2 bytes")
    out = torch.empty(w4_bytes(N, K), dtype=torch.uint8, device=u4packed.device)
    _check(lib().sq_repack_w4(u4packed.data_ptr(), N, K, out.data_ptr(), _stream()))
    return out


def w4a16_bytes(N: int, K: int, group: int) -> int:
    return int(lib().sq_w4a16_bytes(N, K, group))


def repack_w4a16(u4packed: torch.Tensor, N: int, K: int, group: int) -> torch.Tensor:
    """u4packed [N x K/2] (SPEC order) -> the W4A16 GEMV layout (sq_repack_w4a16)."""
    _dev(u4packed, torch.uint8, "u4packed")
    if u4packed.numel() != N * K // 2:
        raise ShapeError(f"u4packed must hold {N * K // 2} bytes")
    out = torch.empty(w4a16_bytes(N, K, group), dtype=torch.uint8, device=u4packed.device)
    _check(lib().sq_repack_w4a16(u4packed.data_ptr(), N, K, group, out.data_ptr(), _stream()))
    return out


def unpack_w4(w: torch.Tensor, N: int, K: int) -> torch.Tensor:
    _dev(w, torch.uint8, "w4")
    out = torch.empty((N, K // 2), dtype=torch.uint8, device=w.device)
    _check(lib().sq_unpack_w4(w.data_ptr(), N, K, out.data_ptr(), _stream()))
    return out


# ------------------------------------------------------------------ row ops
def _gs(gsum, M, K):
    """Optional int32 [M x K/128] activation block sums (see sq_gemm_w4a8)."""
    if gsum is None:
        return 0, 0
    _dev(gsum, torch.int32, "gsum", 2)
    if gsum.shape[0] < M or gsum.shape[1] < K // 128:
        raise ShapeError(f"gsum must be at least [{M} x {K // 128}]")
    return gsum.data_ptr(), _ld(gsum)


def rmsnorm_quant(x, gamma, eps, s, out=None, gsum=None):
    """Pre-norm + per-tensor quant; ``gsum`` (optional) receives the 128-block code sums."""
    _dev(x, torch.float32, "x", 2)
    _dev(gamma, torch.float32, "gamma", 1)
    M, D = x.shape
    out = torch.empty((M, D), dtype=torch.int8, device=x.device) if out is None else out
    _dev(out, torch.int8, "out", 2)
    gp, gl = _gs(gsum, M, D)
    _check(lib().sq_rmsnorm_quant(x.data_ptr(), _ld(x), gamma.data_ptr(), float(eps), float(s), M, D,
                                  out.data_ptr(), _ld(out), gp, gl, _stream()),
           1 + (gsum is not None and D % 16 != 0))
    return out


def rmsnorm_f32(x, gamma, eps, out=None):
    _dev(x, torch.float32, "x", 2)
    M, D = x.shape
    out = torch.empty((M, D), dtype=torch.float32, device=x.device) if out is None else out
    _dev(out, torch.float32, "out", 2)
    _check(lib().sq_rmsnorm_f32(x.data_ptr(), _ld(x), gamma.data_ptr(), float(eps), M, D, out.data_ptr(),
                                _ld(out), _stream()))
    return out


def quantize_f32(x, s, out=None):
    _dev(x, torch.float32, "x", 2)
    M, D = x.shape
    out = torch.empty((M, D), dtype=torch.int8, device=x.device) if out is None else out
    _dev(out, torch.int8, "out", 2)
    _check(lib().sq_quantize_f32(x.data_ptr(), _ld(x), float(s), M, D, out.data_ptr(), _ld(out), _stream()))
    return out


def embed_int8(codes, row_scale, tok, out=None):
    _dev(codes, torch.int8, "codes", 2)
    _dev(tok, torch.int32, "tok", 1)
    M, D = tok.shape[0], codes.shape[1]
    out = torch.empty((M, D), dtype=torch.float32, device=codes.device) if out is None else out
    _check(lib().sq_embed_int8(codes.data_ptr(), row_scale.data_ptr(), tok.data_ptr(), M, D, out.data_ptr(),
                               _stream()))
    return out


def embed_u4(packed, row_scale, tok, D, out=None):
    """4-bit embedding rows: ``packed`` uint8 u4packed [V x D/2]."""
    _dev(packed, torch.uint8, "packed", 2)
    _dev(tok, torch.int32, "tok", 1)
    if packed.shape[1] * 2 != D:
        raise ShapeError(f"packed rows must hold {D} nibbles")
    M = tok.shape[0]
    out = torch.empty((M, D), dtype=torch.float32, device=packed.device) if out is None else out
    _check(lib().sq_embed_u4(packed.data_ptr(), row_scale.data_ptr(), tok.data_ptr(), M, D, out.data_ptr(),
                             _stream()))
    return out


def argmax(logits, out=None):
    _dev(logits, torch.float32, "logits", 2)
    M, N = logits.shape
    out = torch.empty(M, dtype=torch.int32, device=logits.device) if out is None else out
    _check(lib().sq_argmax_f32(logits.data_ptr(), _ld(logits), M, N, out.data_ptr(), _stream()))
    return out


def gate_norm_had_quant(y, gamma, eps, s_y, hadamard=True, out=None):
    _dev(y, torch.float32, "y", 2)
    M, D = y.shape
    out = torch.empty((M, D), dtype=torch.int8, device=y.device) if out is None else out
    _dev(out, torch.int8, "out", 2)
    _check(lib().sq_gate_norm_had_quant(y.data_ptr(), _ld(y), gamma.data_ptr(), float(eps), float(s_y),
                                        int(bool(hadamard)), M, D, out.data_ptr(), _ld(out), _stream()))
    return out


# ------------------------------------------------------------------ projections
_OUT_DTYPE = {EPI_I32: torch.int32, EPI_F32: torch.float32, EPI_QUANT: torch.int8, EPI_RESID: torch.float32}


def _gemm_out(a, N, epi, out):
    M = a.shape[0]
    if out is None:
        if epi == EPI_RESID:
            raise ValueError("EPI_RESID needs the residual tensor as `out`")
        out = torch.empty((M, N), dtype=_OUT_DTYPE[epi], device=a.device)
    _dev(out, _OUT_DTYPE[epi], "out", 2)
    if out.shape[0] != M or out.shape[1] != N:
        raise ShapeError(f"out must be [{M}x{N}], got {tuple(out.shape)}")
    return out


def gemm_w8a8(a, w, alpha, epi=EPI_F32, out=None, col_scale=None):
    _dev(a, torch.int8, "a", 2)
    _dev(w, torch.int8, "w", 2)
    M, K = a.shape
    N = w.shape[0]
    if w.shape[1] != K:
        raise ShapeError(f"w must be [N x {K}]")
    out = _gemm_out(a, N, epi, out)
    _check(lib().sq_gemm_w8a8(a.data_ptr(), _ld(a), w.data_ptr(), alpha.data_ptr(), M, N, K, epi, out.data_ptr(),
                              _ld(out), _opt(col_scale), _stream()))
    return out


def tile_group_scales(s_group):
    """SPEC PerGroup scales [N x G] f32 -> the W4A8 kernel's tiled layout [ceil(N/128)][G][128]."""
    _dev(s_group, torch.float32, "s_group", 2)
    N, G = s_group.shape
    s = s_group.contiguous()
    out = torch.empty(int(lib().sq_group_scale_elems(N, G)), dtype=torch.float32, device=s.device)
    _check(lib().sq_tile_group_scales(s.data_ptr(), N, G, out.data_ptr(), _stream()))
    return out


def gemm_w4a8_splits(M: int, N: int, K: int) -> int:
    """K split of the W4A8 tensor-core kernel for this shape (its f32 summation order)."""
    return int(lib().sq_gemm_w4a8_splits(M, N, K))


def gemm_w4a8(a, w4, w_scale, group, s_a, N, epi=EPI_F32, out=None, col_scale=None):
    """W4A8 projection with SPEC per-group scales; ``w_scale`` in the tiled layout of
    ``tile_group_scales``, ``s_a`` the per-tensor activation scale."""
    _dev(a, torch.int8, "a", 2)
    _dev(w4, torch.uint8, "w4")
    _dev(w_scale, torch.float32, "w_scale")
    M, K = a.shape
    if K % group:
        raise LayoutError(f"group {group} must divide K={K}")
    if w_scale.numel() != int(lib().sq_group_scale_elems(N, K // group)):
        raise LayoutError(f"w_scale must hold the tiled [{N} x {K // group}] group scales")
    if w4.numel() < w4_bytes(N, K):
        raise ShapeError(f"w4 must hold {w4_bytes(N, K)} bytes")
    if epi == EPI_QUANT and (col_scale is None or col_scale.numel() < N):
        raise ShapeError("EPI_QUANT needs col_scale [N]")
    out = _gemm_out(a, N, epi, out)
    _check(lib().sq_gemm_w4a8(a.data_ptr(), _ld(a), w4.data_ptr(), w_scale.data_ptr(), group, float(s_a), M, N, K,
                              epi, out.data_ptr(), _ld(out), _opt(col_scale), _stream()))
    return out


def gemv_w4a16(x, w4, s_group, group, N, out=None, resid=False, norm_w=None, eps=1e-5, conv=None):
    """W4A16 projection: x f32 [M x K] (rounded to bf16 on load; RMS-normalised with norm_w
    first when given), w4 in the sq_repack_w4a16 layout, s_group f32 [N x K/group]; out f32
    [M x N] (+= when resid).  ``conv`` = (w [C x Kc], bias [C], c0, cache [M x (Kc-1) x C],
    cache_in, conv_out [M x C]) fuses the T = 1 causal-conv update of output columns
    c0 .. c0+C-1 into the epilogue (sq_gemv_w4a16_conv)."""
    _dev(x, torch.float32, "x", 2)
    _dev(w4, torch.uint8, "w4")
    M, K = x.shape
    if w4.numel() < w4a16_bytes(N, K, group):
        raise ShapeError(f"w4 must hold {w4a16_bytes(N, K, group)} bytes")
    _dev(s_group, torch.float32, "s_group", 2)
    if tuple(s_group.shape) != (N, K // group):
        raise ShapeError(f"s_group must be [{N} x {K // group}]")
    if norm_w is not None:
        _dev(norm_w, torch.float32, "norm_w", 1)
        if norm_w.numel() != K:
            raise ShapeError(f"norm_w must hold {K} values")
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=x.device)
    _dev(out, torch.float32, "out", 2)
    if conv is None:
        _check(lib().sq_gemv_w4a16(x.data_ptr(), _ld(x), norm_w.data_ptr() if norm_w is not None else None,
                                   float(eps), w4.data_ptr(), s_group.data_ptr(), group, M, N, K, out.data_ptr(),
                                   _ld(out), int(bool(resid)), _stream()))
        return out
    cw, cb, c0, cache, cache_in, cout = conv
    _dev(cw, torch.float32, "conv w", 2)
    _dev(cache, torch.float32, "conv cache")
    _dev(cout, torch.float32, "conv out", 2)
    Cc, Kc = cw.shape
    _need(cache, M * (Kc - 1) * Cc, "conv cache [M x (K-1) x C]")
    _rows(cout, M, "conv out")
    ep = _lib.ConvEpilogue(cw.data_ptr(), cb.data_ptr(), Kc, int(c0), Cc, cache.data_ptr(), int(bool(cache_in)),
                           cout.data_ptr(), _ld(cout))
    _check(lib().sq_gemv_w4a16_conv(x.data_ptr(), _ld(x), norm_w.data_ptr() if norm_w is not None else None,
                                    float(eps), w4.data_ptr(), s_group.data_ptr(), group, M, N, K, out.data_ptr(),
                                    _ld(out), int(bool(resid)), C.byref(ep), _stream()))
    return out


# ------------------------------------------------------------------ conv
def conv1d_int8(x, w, bias, s_in, s_out, B, T, cache, cache_in=False, out=None):
    _dev(x, torch.int8, "x", 2)
    _dev(cache, torch.int8, "cache")
    C_, Kc = w.shape
    _rows(x, B * T, "x")
    _need(cache, B * (Kc - 1) * C_, "cache [B x (K-1) x C]")
    out = torch.empty((B * T, C_), dtype=torch.int8, device=x.device) if out is None else out
    _rows(out, B * T, "out")
    _check(lib().sq_conv1d_int8(x.data_ptr(), _ld(x), w.data_ptr(), bias.data_ptr(), s_in.data_ptr(),
                                s_out.data_ptr(), B, T, C_, Kc, cache.data_ptr(), int(bool(cache_in)),
                                out.data_ptr(), _ld(out), _stream()),
           1 if (Kc == 4 and C_ % 4 == 0 and _ld(x) % 4 == 0 and _ld(out) % 4 == 0 and x.data_ptr() % 4 == 0
                 and out.data_ptr() % 4 == 0) else 1 + (Kc > 1))   # 4-channel kernel writes the cache itself
    return out


def conv1d_update_int8(x, w, bias, s_in, s_out, cache, out=None):
    _dev(x, torch.int8, "x", 2)
    _dev(cache, torch.int8, "cache")
    B = x.shape[0]
    C_, Kc = w.shape
    _need(cache, B * (Kc - 1) * C_, "cache [B x (K-1) x C]")
    out = torch.empty((B, C_), dtype=torch.int8, device=x.device) if out is None else out
    _rows(out, B, "out")
    _check(lib().sq_conv1d_update_int8(x.data_ptr(), _ld(x), w.data_ptr(), bias.data_ptr(), s_in.data_ptr(),
                                       s_out.data_ptr(), B, C_, Kc, cache.data_ptr(), out.data_ptr(), _ld(out),
                                       _stream()))
    return out


def conv1d_f32(x, w, bias, B, T, cache, cache_in=False, out=None):
    _dev(x, torch.float32, "x", 2)
    _dev(cache, torch.float32, "cache")
    C_, Kc = w.shape
    _rows(x, B * T, "x")
    _need(cache, B * (Kc - 1) * C_, "cache [B x (K-1) x C]")
    out = torch.empty((B * T, C_), dtype=torch.float32, device=x.device) if out is None else out
    _rows(out, B * T, "out")
    _check(lib().sq_conv1d_f32(x.data_ptr(), _ld(x), w.data_ptr(), bias.data_ptr(), B, T, C_, Kc, cache.data_ptr(),
                               int(bool(cache_in)), out.data_ptr(), _ld(out), _stream()), 1 + (Kc > 1 and T > 1))
    return out


# ------------------------------------------------------------------ scans
def mamba2_params(n_heads, head_dim, d_state, n_groups, head_group, A, D, dt_bias, s_dt=1.0, s_z=1.0,
                  s_x=None, s_B=None, s_C=None, s_h=None) -> _lib.Mamba2Params:
    """Build the parameter struct; keeps no reference to the tensors (caller owns them)."""
    return _lib.Mamba2Params(n_heads, head_dim, d_state, n_groups, head_group.data_ptr(), A.data_ptr(),
                             D.data_ptr(), dt_bias.data_ptr(), float(s_dt), float(s_z), _opt(s_x), _opt(s_B),
                             _opt(s_C), _opt(s_h))


def mamba2_decode_params(ssm: _lib.Mamba2Params, conv_w, conv_b, conv_s_in, conv_s_out, norm_w, eps, s_y,
                         hadamard=True) -> _lib.Mamba2DecodeParams:
    return _lib.Mamba2DecodeParams(ssm, int(conv_w.shape[1]), conv_w.data_ptr(), conv_b.data_ptr(),
                                   conv_s_in.data_ptr(), conv_s_out.data_ptr(), norm_w.data_ptr(), float(eps),
                                   float(s_y), int(bool(hadamard)))


def mamba2_decode_ws_bytes(p, B) -> int:
    return int(lib().sq_mamba2_decode_ws_bytes(C.byref(p), B))


def mamba2_decode_step_int8(p, B, zx, conv_cache, state, yq=None, y=None, ws=None, gsum=None):
    """Mamba2 decode step, SSM half of a block (conv update + int8 state update + gated
    norm + FWHT + quant).  zx int8 [B x in_proj_out] (z|x|B|C|dt codes); conv_cache int8
    [B x (K-1) x conv_dim]; state int8 [B x nh x P x N] (both updated in place).  Returns
    yq int8 [B x d_inner]; ``y`` (f32 [B x d_inner], gated SSM output) and ``ws`` (uint8,
    mamba2_decode_ws_bytes) are workspaces, allocated when not given."""
    _dev(zx, torch.int8, "zx", 2)
    _dev(conv_cache, torch.int8, "conv_cache")
    _dev(state, torch.int8, "state")
    di = p.ssm.n_heads * p.ssm.head_dim
    conv_dim = di + 2 * p.ssm.n_groups * p.ssm.d_state
    _rows(zx, B, "zx")
    _need(state, B * p.ssm.n_heads * p.ssm.head_dim * p.ssm.d_state, "state [B x nh x P x N]")
    _need(conv_cache, B * (p.conv_kernel - 1) * conv_dim, "conv_cache [B x (K-1) x conv_dim]")
    if yq is None:
        yq = torch.empty((B, di), dtype=torch.int8, device=zx.device)
    if y is None:
        y = torch.empty((B, di), dtype=torch.float32, device=zx.device)
    nbytes = mamba2_decode_ws_bytes(p, B)
    if ws is None:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=zx.device)
    if ws.numel() * ws.element_size() < nbytes:
        raise ShapeError(f"decode workspace needs {nbytes} bytes")
    _dev(yq, torch.int8, "yq", 2)
    _dev(y, torch.float32, "y", 2)
    gp, gl = _gs(gsum, B, di)
    _check(lib().sq_mamba2_decode_step_int8(C.byref(p), B, zx.data_ptr(), _ld(zx), conv_cache.data_ptr(),
                                            state.data_ptr(), ws.data_ptr(), y.data_ptr(), _ld(y), yq.data_ptr(),
                                            _ld(yq), gp, gl, _stream()),
           int(lib().sq_mamba2_decode_launches(C.byref(p), B, int(gsum is not None))))
    return yq


def mamba1_decode_params(ssm: _lib.Mamba1Params, conv_w, conv_b, conv_s_in, conv_s_out, dt_rank, xproj_w,
                         xproj_alpha, xproj_cs, dtproj_w, dtproj_alpha, dtproj_cs, norm_w, eps, s_y,
                         hadamard=True) -> _lib.Mamba1DecodeParams:
    """Parameter struct of the one-launch Mamba1 W8A8 decode step; keeps no tensor references."""
    return _lib.Mamba1DecodeParams(ssm, int(conv_w.shape[1]), conv_w.data_ptr(), conv_b.data_ptr(),
                                   conv_s_in.data_ptr(), conv_s_out.data_ptr(), int(dt_rank), xproj_w.data_ptr(),
                                   xproj_alpha.data_ptr(), xproj_cs.data_ptr(), dtproj_w.data_ptr(),
                                   dtproj_alpha.data_ptr(), dtproj_cs.data_ptr(), norm_w.data_ptr(), float(eps),
                                   float(s_y), int(bool(hadamard)))


def mamba1_decode_ws_bytes(p, B) -> int:
    return int(lib().sq_mamba1_decode_ws_bytes(C.byref(p), B))


def mamba1_decode_step_int8(p, B, zx, conv_cache, state, ws, yq=None):
    """Mamba1 W8A8 decode step, SSM half of a block in one launch (conv update, x_proj, dt_proj,
    int8 scan step, gated norm + FWHT + quant).  zx int8 [B x 2*d_inner] (z | x); conv_cache int8
    [B x (K-1) x d_inner] and state int8 [B x d_inner x 16] are updated in place; ``ws`` (uint8,
    mamba1_decode_ws_bytes) must have been zero-filled once (grid-barrier counters).  Returns
    yq int8 [B x d_inner]."""
    _dev(zx, torch.int8, "zx", 2)
    _dev(conv_cache, torch.int8, "conv_cache")
    _dev(state, torch.int8, "state")
    di = p.ssm.d_inner
    _rows(zx, B, "zx")
    _need(state, B * di * p.ssm.d_state, "state [B x d_inner x N]")
    _need(conv_cache, B * (p.conv_kernel - 1) * di, "conv_cache [B x (K-1) x d_inner]")
    if yq is None:
        yq = torch.empty((B, di), dtype=torch.int8, device=zx.device)
    _dev(yq, torch.int8, "yq", 2)
    nbytes = mamba1_decode_ws_bytes(p, B)
    if ws is None or ws.numel() * ws.element_size() < nbytes:
        raise ShapeError(f"Mamba1 decode workspace needs {nbytes} zero-initialised bytes")
    _check(lib().sq_mamba1_decode_step_int8(C.byref(p), B, zx.data_ptr(), _ld(zx), conv_cache.data_ptr(),
                                            state.data_ptr(), ws.data_ptr(), yq.data_ptr(), _ld(yq), _stream()), 1)
    return yq


def mamba1_layer_params(ln_w, eps, s_u, d_model, in_w, in_alpha, in_cs, out_w, out_alpha) -> _lib.Mamba1LayerParams:
    return _lib.Mamba1LayerParams(ln_w.data_ptr(), float(eps), float(s_u), int(d_model), in_w.data_ptr(),
                                  in_alpha.data_ptr(), in_cs.data_ptr(), out_w.data_ptr(), out_alpha.data_ptr())


def mamba1_decode_layer_int8(p, lp, B, h, conv_cache, state, ws):
    """A whole Mamba1 W8A8 decode layer in one launch: h f32 [B x d_model] (the residual stream,
    updated in place: pre-norm + in_proj + SSM half + out_proj residual add); ``ws`` as
    mamba1_decode_step_int8's (zeroed once)."""
    _dev(h, torch.float32, "h", 2)
    _dev(conv_cache, torch.int8, "conv_cache")
    _dev(state, torch.int8, "state")
    _rows(h, B, "h")
    di = p.ssm.d_inner
    _need(state, B * di * p.ssm.d_state, "state [B x d_inner x N]")
    _need(conv_cache, B * (p.conv_kernel - 1) * di, "conv_cache [B x (K-1) x d_inner]")
    nbytes = mamba1_decode_ws_bytes(p, B)
    if ws is None or ws.numel() * ws.element_size() < nbytes:
        raise ShapeError(f"Mamba1 decode workspace needs {nbytes} zero-initialised bytes")
    _check(lib().sq_mamba1_decode_layer_int8(C.byref(p), C.byref(lp), B, h.data_ptr(), _ld(h),
                                             conv_cache.data_ptr(), state.data_ptr(), ws.data_ptr(), _stream()), 1)
    return h


def mamba1_params(d_inner, d_state, A, D, dt_bias, s_dt, s_z, s_B, s_C, s_x, s_h) -> _lib.Mamba1Params:
    return _lib.Mamba1Params(d_inner, d_state, A.data_ptr(), D.data_ptr(), dt_bias.data_ptr(), float(s_dt),
                             float(s_z), float(s_B), float(s_C), s_x.data_ptr(), s_h.data_ptr())


def ssd_scan_int8(p, B, T, x, Bm, Cm, dt, z, state, state_in, y, chunk=256):
    for n, t in (("x", x), ("B", Bm), ("C", Cm), ("dt", dt), ("z", z)):
        _dev(t, torch.int8, n, 2)
    _dev(state, torch.int8, "state")
    _need(state, B * p.n_heads * p.head_dim * p.d_state, "state [B x nh x P x N]")
    _dev(y, torch.float32, "y", 2)
    _check(lib().sq_ssd_scan_int8(C.byref(p), B, T, x.data_ptr(), _ld(x), Bm.data_ptr(), Cm.data_ptr(), _ld(Bm),
                                  dt.data_ptr(), _ld(dt), z.data_ptr(), _ld(z), state.data_ptr(),
                                  int(bool(state_in)), y.data_ptr(), _ld(y), int(chunk), _stream()))
    return y


def state_update_int8(p, B, x, Bm, Cm, dt, z, state, y):
    for n, t in (("x", x), ("B", Bm), ("C", Cm), ("dt", dt), ("z", z)):
        _dev(t, torch.int8, n, 2)
    _dev(state, torch.int8, "state")
    _need(state, B * p.n_heads * p.head_dim * p.d_state, "state [B x nh x P x N]")
    _dev(y, torch.float32, "y", 2)
    _check(lib().sq_state_update_int8(C.byref(p), B, x.data_ptr(), _ld(x), Bm.data_ptr(), Cm.data_ptr(), _ld(Bm),
                                      dt.data_ptr(), _ld(dt), z.data_ptr(), _ld(z), state.data_ptr(), y.data_ptr(),
                                      _ld(y), _stream()))
    return y


def ssd_scan_f32(p, B, T, x, Bm, Cm, dt, z, state, state_in, y):
    for n, t in (("x", x), ("B", Bm), ("C", Cm), ("dt", dt), ("z", z)):
        _dev(t, torch.float32, n, 2)
    _dev(state, torch.float32, "state")
    _need(state, B * p.n_heads * p.head_dim * p.d_state, "state [B x nh x P x N]")
    _check(lib().sq_ssd_scan_f32(C.byref(p), B, T, x.data_ptr(), _ld(x), Bm.data_ptr(), Cm.data_ptr(), _ld(Bm),
                                 dt.data_ptr(), _ld(dt), z.data_ptr(), _ld(z), state.data_ptr(), int(bool(state_in)),
                                 y.data_ptr(), _ld(y), _stream()))
    return y


def selective_scan_int8(p, B, T, x, dt, BC, z, state, state_in, y, ws=None):
    """Mamba1 int8 selective scan; long prompts run the time-chunked two-pass form in a
    workspace of sq_selective_scan_int8_ws_bytes (allocated here unless given)."""
    for n, t in (("x", x), ("dt", dt), ("BC", BC), ("z", z)):
        _dev(t, torch.int8, n, 2)
    _dev(state, torch.int8, "state")
    _need(state, B * p.d_inner * p.d_state, "state [B x d_inner x N]")
    nb = int(lib().sq_selective_scan_int8_ws_bytes(C.byref(p), B, T))
    if nb > 0 and ws is None:
        ws = torch.empty(nb, dtype=torch.uint8, device=x.device)
    if ws is not None and ws.numel() * ws.element_size() < nb:
        raise ShapeError(f"selective scan workspace needs {nb} bytes")
    _check(lib().sq_selective_scan_int8(C.byref(p), B, T, x.data_ptr(), _ld(x), dt.data_ptr(), _ld(dt),
                                        BC.data_ptr(), _ld(BC), z.data_ptr(), _ld(z), state.data_ptr(),
                                        int(bool(state_in)), y.data_ptr(), _ld(y),
                                        ws.data_ptr() if nb > 0 else None, _stream()),
           2 if nb > 0 else 1)
    return y


def selective_scan_f32(p, B, T, x, dt, BC, z, state, state_in, y):
    """Mamba1 W4A16 scan (float operands, f32 state)."""
    for n, t in (("x", x), ("dt", dt), ("BC", BC), ("z", z), ("y", y)):
        _dev(t, torch.float32, n, 2)
    _dev(state, torch.float32, "state")
    _need(state, B * p.d_inner * p.d_state, "state [B x d_inner x N]")
    _check(lib().sq_selective_scan_f32(C.byref(p), B, T, x.data_ptr(), _ld(x), dt.data_ptr(), _ld(dt),
                                       BC.data_ptr(), _ld(BC), z.data_ptr(), _ld(z), state.data_ptr(),
                                       int(bool(state_in)), y.data_ptr(), _ld(y), _stream()))
    return y


# ------------------------------------------------------------------ SPEC float ops
def discretize_f32(dt_raw, dt_bias, A):
    """Δ = softplus(Δ_raw + dt_bias), Ȧ = exp(Δ·A).  dt_raw [M×H];
    A [H] (Mamba2) or [H×N] (Mamba1) → (Ȧ [M×H] or [M×H×N], Δ [M×H])."""
    _dev(dt_raw, torch.float32, "dt_raw", 2)
    _dev(dt_bias, torch.float32, "dt_bias", 1)
    _dev(A, torch.float32, "A")
    M, H = dt_raw.shape
    N = 1 if A.dim() == 1 else A.shape[1]
    if A.shape[0] != H or dt_bias.shape[0] != H:
        raise ShapeError(f"A / dt_bias must have {H} rows")
    dA = torch.empty((M, H) if A.dim() == 1 else (M, H, N), dtype=torch.float32, device=dt_raw.device)
    delta = torch.empty((M, H), dtype=torch.float32, device=dt_raw.device)
    _check(lib().sq_discretize_f32(dt_raw.data_ptr(), _ld(dt_raw), dt_bias.data_ptr(), A.contiguous().data_ptr(),
                                   M, H, N, dA.data_ptr(), delta.data_ptr(), _stream()))
    return dA, delta


def selective_scan2_pre_f32(p, B, T, x, dA, delta, Bm, Cm, z, state, state_in, y):
    """Mamba2 recurrence on precomputed Ȧ / Δ [B·T×nh]; z None = ungated."""
    for n, t in (("x", x), ("dA", dA), ("delta", delta), ("B", Bm), ("C", Cm), ("y", y)):
        _dev(t, torch.float32, n, 2)
    _dev(state, torch.float32, "state")
    if dA.stride(0) != delta.stride(0) or Bm.stride(0) != Cm.stride(0):
        raise LayoutError("dA/delta and B/C must share row strides")
    if state.numel() != B * p.n_heads * p.head_dim * p.d_state:
        raise ShapeError("state must be [B x nh x P x N]")
    _check(lib().sq_selective_scan2_pre_f32(C.byref(p), B, T, x.data_ptr(), _ld(x), dA.data_ptr(), delta.data_ptr(),
                                            _ld(dA), Bm.data_ptr(), Cm.data_ptr(), _ld(Bm), _opt(z),
                                            0 if z is None else _ld(z), state.data_ptr(), int(bool(state_in)),
                                            y.data_ptr(), _ld(y), _stream()))
    return y


def selective_scan1_pre_f32(p, B, T, x, dA, delta, Bm, Cm, z, state, state_in, y):
    """Mamba1 recurrence on precomputed Ȧ [B·T×d×N] / Δ [B·T×d]; z None = ungated."""
    for n, t in (("x", x), ("delta", delta), ("B", Bm), ("C", Cm), ("y", y)):
        _dev(t, torch.float32, n, 2)
    _dev(dA, torch.float32, "dA", 3)
    _dev(state, torch.float32, "state")
    if Bm.stride(0) != Cm.stride(0):
        raise LayoutError("B and C must share a row stride")
    if state.numel() != B * p.d_inner * p.d_state:
        raise ShapeError("state must be [B x d_inner x N]")
    _check(lib().sq_selective_scan1_pre_f32(C.byref(p), B, T, x.data_ptr(), _ld(x), dA.data_ptr(), delta.data_ptr(),
                                            _ld(delta), Bm.data_ptr(), Cm.data_ptr(), _ld(Bm), _opt(z),
                                            0 if z is None else _ld(z), state.data_ptr(), int(bool(state_in)),
                                            y.data_ptr(), _ld(y), _stream()))
    return y

