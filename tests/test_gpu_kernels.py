"""GPU parity: every C-ABI kernel vs the CPU oracle on the same seeded inputs.

Bars (north_star): int32 accumulators, weight codes and packing bit-exact; requantised
int8 activations / cached state within 1 quantization step (mismatch fractions
reported and bounded); float outputs within the stated relative tolerance.
"""
import numpy as np
import pytest
import torch

from oracle import hadamard as ohad
from oracle import qblock as oq
from oracle import ssm_block as osb
from oracle.quantizer import quantize_codes
from oracle.tensor_core import int_gemm, pack_u4, unpack_u4

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2503_22879_b200 import ops
    return ops


def _rng(*s):
    from oracle.tensor_core import make_rng
    return make_rng(1234, *s)


def code_diff(a, b):
    d = np.abs(np.asarray(a, np.int32) - np.asarray(b, np.int32))
    return int(d.max(initial=0)), float((d > 0).mean()) if d.size else 0.0


# K % 128 != 0 with M > 16 runs the mma.sync kernel, the rest the tcgen05 kernels
@pytest.mark.parametrize("M,N,K", [(1, 128, 64), (64, 18560 // 8, 4096), (37, 300, 160), (256, 1024, 512),
                                   (64, 4096, 8192), (200, 2560, 5120), (1, 5120, 256), (1, 5120, 160),
                                   (3, 192, 5120), (8, 1000, 2560), (5, 10240, 2560)])
def test_gemm_w8a8_exact(cuda, M, N, K):
    ops = _ops()
    r = _rng(1, M, N)
    a = r.integers(-128, 128, (M, K)).astype(np.int8)
    w = r.integers(-127, 128, (N, K)).astype(np.int8)
    alpha = r.uniform(1e-4, 1e-2, N).astype(np.float32)
    cs = r.uniform(0.05, 0.2, N).astype(np.float32)
    ta, tw, tal, tcs = (torch.as_tensor(x, device=cuda) for x in (a, w, alpha, cs))
    acc = int_gemm(a, w.T)
    got = ops.gemm_w8a8(ta, tw, tal, ops.EPI_I32).cpu().numpy()
    assert np.array_equal(got, acc), "int32 accumulators must be bit-exact"
    y = (acc.astype(np.float32) * alpha[None]).astype(np.float32)
    gy = ops.gemm_w8a8(ta, tw, tal, ops.EPI_F32).cpu().numpy()
    assert np.array_equal(gy, y)
    q = quantize_codes(y, cs[None], 8)
    gq = ops.gemm_w8a8(ta, tw, tal, ops.EPI_QUANT, col_scale=tcs).cpu().numpy()
    assert np.array_equal(gq, q)
    res = r.standard_normal((M, N)).astype(np.float32)
    tres = torch.as_tensor(res, device=cuda)
    ops.gemm_w8a8(ta, tw, tal, ops.EPI_RESID, out=tres)
    assert np.array_equal(tres.cpu().numpy(), (res + y).astype(np.float32))


def _same(got, want, what):
    """Exact equality with a diagnostic of where the results differ."""
    d = got != want
    if d.any():
        r, c = np.nonzero(d)
        raise AssertionError(f"{what}: {d.sum()} of {d.size} differ; rows {np.unique(r)[:10]} (x{len(np.unique(r))}), "
                             f"col tiles {np.unique(c // 128)}; first got {got[r[0], c[0]]} want {want[r[0], c[0]]}")


def _w4a8_case(r, M, N, K, group, cuda, unit_scales=False):
    ops = _ops()
    from paper_2503_22879_b200.ssm_block import pack_u4_host
    a = r.integers(-128, 128, (M, K)).astype(np.int8)
    codes = r.integers(-8, 8, (N, K)).astype(np.int8)
    if unit_scales:
        sgrp = np.ones((N, K // group), np.float32)
    else:
        sgrp = (r.uniform(1e-3, 1e-2, (N, K // group)) * np.exp(r.uniform(-3, 3, (N, K // group)))).astype(np.float32)
    ql = oq.QLinear("w4a8", codes, s_group=sgrp, group=group)
    packed = pack_u4_host(codes)
    assert np.array_equal(packed, pack_u4(codes)), "product packing == oracle packing"
    tw = ops.repack_w4(torch.as_tensor(packed, device=cuda), N, K)
    assert np.array_equal(ops.unpack_w4(tw, N, K).cpu().numpy(), packed)
    tws = ops.tile_group_scales(torch.as_tensor(sgrp, device=cuda))
    return a, ql, tw, tws


@pytest.mark.parametrize("M,N,K,group", [(64, 384, 4096, 128), (3, 256, 256, 32), (16, 130, 8192, 128),
                                         (64, 4096, 8192, 128), (64, 18560, 4096, 128), (300, 640, 1024, 128),
                                         (1, 4096, 8192, 128), (33, 1000, 2560, 128), (5, 5120, 160, 32)])
def test_gemm_w4a8_exact(cuda, M, N, K, group):
    """W4A8 with SPEC per-group float scales (LEDGER G11): the int32 per-group partials are exact
    (unit scales: y == the int32 total), and the promoted f32 sum follows the oracle's order
    (ascending groups per K split, splits in order) bit for bit, as do the requantized codes
    and the residual add."""
    ops = _ops()
    r = _rng(2, M, N)
    a, ql1, tw, tws1 = _w4a8_case(r, M, N, K, group, cuda, unit_scales=True)
    ta = torch.as_tensor(a, device=cuda)
    acc = int_gemm(a, ql1.codes.T)
    assert np.abs(acc).max() < 2 ** 24
    gy = ops.gemm_w4a8(ta, tw, tws1, group, 1.0, N, ops.EPI_F32).cpu().numpy()
    _same(gy, acc.astype(np.float32), "int32 partials (unit scales)")
    a, ql, tw, tws = _w4a8_case(r, M, N, K, group, cuda)
    ta = torch.as_tensor(a, device=cuda)
    s_a = np.float32(0.0173)
    splits = ops.gemm_w4a8_splits(M, N, K) if group == 128 else 1
    y, _ = oq.qlinear_a8(a, ql, s_a, splits=splits)
    gy = ops.gemm_w4a8(ta, tw, tws, group, s_a, N, ops.EPI_F32).cpu().numpy()
    _same(gy, y, f"F32 (splits={splits})")
    cs = r.uniform(0.5, 2.0, N).astype(np.float32) * np.float32(np.abs(y).max() / 127)
    gq = ops.gemm_w4a8(ta, tw, tws, group, s_a, N, ops.EPI_QUANT, col_scale=torch.as_tensor(cs, device=cuda))
    _same(gq.cpu().numpy(), quantize_codes(y, cs[None], 8), "QUANT")
    res = r.standard_normal((M, N)).astype(np.float32)
    tres = torch.as_tensor(res, device=cuda)
    ops.gemm_w4a8(ta, tw, tws, group, s_a, N, ops.EPI_RESID, out=tres)
    _same(tres.cpu().numpy(), (res + y).astype(np.float32), "RESID")


@pytest.mark.parametrize("M,N,K,group", [(1, 18560, 4096, 128), (1, 4096, 8192, 128), (3, 512, 8192, 128),
                                         (8, 1000, 4096, 64), (5, 100, 256, 16), (11, 33, 192, 32),
                                         (16, 200, 160, 32)])
def test_gemv_w4a16(cuda, M, N, K, group):
    """W4A16 GEMV (bf16 activations, f32 accumulation) vs the oracle (x rounded to bf16 the
    same way): mma.sync fragment layout for K % 64 == 0, group 64 / 128 (ragged N, several
    token passes, one or two quads per group), row-major fallback for groups 16 / 32 and K = 160."""
    ops = _ops()
    from paper_2503_22879_b200.ssm_block import pack_u4_host
    r = _rng(3, M, N)
    x = r.standard_normal((M, K)).astype(np.float32)
    codes = r.integers(-8, 8, (N, K)).astype(np.int8)
    sgrp = r.uniform(1e-3, 1e-2, (N, K // group)).astype(np.float32)
    ql = oq.QLinear("w4a16", codes, s_group=sgrp, group=group)
    ref = oq.qlinear_a16(x, ql)
    tw = ops.repack_w4a16(torch.as_tensor(pack_u4_host(codes), device=cuda), N, K, group)
    got = ops.gemv_w4a16(torch.as_tensor(x, device=cuda), tw, torch.as_tensor(sgrp, device=cuda), group, N)
    got = got.cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max() + 1e-6
    # fused RMSNorm of the input rows (the block's gated norm / the model's pre-norm)
    gam = r.uniform(0.5, 1.5, K).astype(np.float32)
    refn = oq.qlinear_a16(osb.rmsnorm(x, gam), ql)
    gotn = ops.gemv_w4a16(torch.as_tensor(x, device=cuda), tw, torch.as_tensor(sgrp, device=cuda), group, N,
                          norm_w=torch.as_tensor(gam, device=cuda)).cpu().numpy()
    assert np.abs(gotn - refn).max() <= 2e-5 * np.abs(refn).max() + 1e-6
    # resid accumulates in place
    base = r.standard_normal((M, N)).astype(np.float32)
    tb = torch.as_tensor(base, device=cuda)
    ops.gemv_w4a16(torch.as_tensor(x, device=cuda), tw, torch.as_tensor(sgrp, device=cuda), group, N, out=tb,
                   resid=True)
    assert np.abs(tb.cpu().numpy() - (base + got)).max() <= 1e-6 * np.abs(base + got).max() + 1e-6


@pytest.mark.parametrize("M,N,K,group", [(1, 1280, 512, 128), (3, 1000, 512, 64), (9, 1280, 256, 128),
                                          (2, 1280, 160, 32)])
def test_gemv_w4a16_conv_epilogue(cuda, M, N, K, group):
    """The T = 1 conv update fused into the W4A16 GEMV epilogue (sq_gemv_w4a16_conv) equals the
    GEMV followed by sq_conv1d_f32 bit for bit (GEMV output, conv output, shifted cache), on the
    mma.sync path (one and two token passes) and the row-major fallback (separate conv launch)."""
    ops = _ops()
    from paper_2503_22879_b200.ssm_block import pack_u4_host
    r = _rng(9, M, N)
    x = torch.as_tensor(r.standard_normal((M, K)).astype(np.float32), device=cuda)
    codes = r.integers(-8, 8, (N, K)).astype(np.int8)
    sgrp = torch.as_tensor(r.uniform(1e-3, 1e-2, (N, K // group)).astype(np.float32), device=cuda)
    tw = ops.repack_w4a16(torch.as_tensor(pack_u4_host(codes), device=cuda), N, K, group)
    c0, C, Kc = 200, 640, 4
    cw = torch.as_tensor(r.standard_normal((C, Kc)).astype(np.float32), device=cuda)
    cb = torch.as_tensor(r.standard_normal(C).astype(np.float32), device=cuda)
    cache = torch.as_tensor(r.standard_normal((M, Kc - 1, C)).astype(np.float32), device=cuda)
    ref_out = ops.gemv_w4a16(x, tw, sgrp, group, N)
    ref_cache = cache.clone()
    ref_conv = ops.conv1d_f32(ref_out[:, c0:c0 + C], cw, cb, M, 1, ref_cache, True)
    cache2 = cache.clone()
    conv_out = torch.empty((M, C), device=cuda)
    out = ops.gemv_w4a16(x, tw, sgrp, group, N, conv=(cw, cb, c0, cache2, True, conv_out))
    torch.cuda.synchronize()
    assert torch.equal(out, ref_out)
    assert torch.equal(conv_out, ref_conv)
    assert torch.equal(cache2, ref_cache)


@pytest.mark.parametrize("M,D", [(5, 256), (64, 4096), (3, 2560)])
def test_rmsnorm_quant(cuda, M, D):
    ops = _ops()
    r = _rng(4, M, D)
    x = (r.standard_normal((M, D)) * np.exp(r.uniform(-2, 2, D))).astype(np.float32)
    g = (1 + 0.1 * r.standard_normal(D)).astype(np.float32)
    s = np.float32(np.abs(osb.rmsnorm(x, g)).max() / 127)
    ref = quantize_codes(osb.rmsnorm(x, g), s, 8)
    gs = torch.zeros((M, D // 128), dtype=torch.int32, device=cuda) if D % 128 == 0 else None
    got = ops.rmsnorm_quant(torch.as_tensor(x, device=cuda), torch.as_tensor(g, device=cuda), 1e-5, s,
                            gsum=gs).cpu().numpy()
    mx, frac = code_diff(got, ref)
    assert mx <= 1 and frac < 1e-3
    if gs is not None:   # block sums of exactly the codes written
        assert np.array_equal(gs.cpu().numpy(), got.astype(np.int32).reshape(M, -1, 128).sum(-1))


@pytest.mark.parametrize("M,D,had", [(4, 512, True), (64, 8192, True), (8, 5120, True), (8, 512, False),
                                     (300, 5120, True), (45, 3072, True), (1, 1024, True), (5, 15360, True)])
def test_gate_norm_had_quant(cuda, M, D, had):
    ops = _ops()
    r = _rng(5, M, D)
    y = (r.standard_normal((M, D)) * np.exp(r.uniform(-1, 1, D))).astype(np.float32)
    g = (1 + 0.1 * r.standard_normal(D)).astype(np.float32)
    rn = osb.rmsnorm(y, g)
    t = ohad.fwht_blocked(rn) if had else rn
    s = np.float32(np.abs(t).max() / 127)
    ref = quantize_codes(t, s, 8)
    got = ops.gate_norm_had_quant(torch.as_tensor(y, device=cuda), torch.as_tensor(g, device=cuda), 1e-5, s,
                                  had).cpu().numpy()
    mx, frac = code_diff(got, ref)
    assert mx <= 1 and frac < 1e-3


@pytest.mark.parametrize("T", [150, 2])   # T < K-1: the new cache window keeps old entries
def test_conv1d_prefill_and_update(cuda, T):
    ops = _ops()
    r = _rng(6, T)
    B, C, K = 3, 384, 4
    x = r.integers(-128, 128, (B * T, C)).astype(np.int8)
    w = (r.standard_normal((C, K)) * 0.3).astype(np.float32)
    b = (r.standard_normal(C) * 0.05).astype(np.float32)
    s_in = r.uniform(0.01, 0.05, C).astype(np.float32)
    s_out = r.uniform(0.01, 0.05, C).astype(np.float32)
    qb = oq.QBlock(None, "W8A8", None, None, w, b, None, None, None, None, conv_in_scale=s_in, conv_out_scale=s_out)
    qb.dims = osb.Dims("mamba2", 8, 8, 8, 1, 8, 1, K)
    cache0 = r.integers(-128, 128, (B, C, K - 1)).astype(np.int8)
    refs, caches = [], []
    for bi in range(B):
        o, c = oq._conv_a8(x[bi * T:(bi + 1) * T], qb, cache0[bi])
        refs.append(o)
        caches.append(c)
    ref = np.concatenate(refs)
    t = lambda a: torch.as_tensor(a, device=cuda)
    tcache = t(np.ascontiguousarray(cache0.transpose(0, 2, 1)))
    got = ops.conv1d_int8(t(x), t(w), t(b), t(s_in), t(s_out), B, T, tcache, True).cpu().numpy()
    mx, frac = code_diff(got, ref)
    assert mx <= 1 and frac < 1e-3
    assert np.array_equal(tcache.cpu().numpy(), np.stack(caches).transpose(0, 2, 1))
    # decode update: one more token per sequence
    xn = r.integers(-128, 128, (B, C)).astype(np.int8)
    refn = np.concatenate([oq._conv_a8(xn[bi:bi + 1], qb, caches[bi])[0] for bi in range(B)])
    gotn = ops.conv1d_update_int8(t(xn), t(w), t(b), t(s_in), t(s_out), tcache).cpu().numpy()
    mx, frac = code_diff(gotn, refn)
    assert mx <= 1 and frac < 1e-2


def _tiny_block(profile, variant="mamba2", seed=0):
    from oracle import pipeline as opl
    if variant == "mamba2":
        d = osb.Dims("mamba2", 256, 512, 64, 8, 64, 2, 4)
    else:
        d = osb.Dims("mamba1", 256, 512, 16, 1, 512, 1, 4, dt_rank=32)
    fm = opl.cmd_gen_toy(d, 1, seed=seed)
    toks = opl.calib_tokens(512, 2, 64, seed)
    stats = opl.collect_stats(fm, toks)
    qb = opl.quantize_block(fm.blocks[0], stats[0], profile)
    u = osb.rmsnorm(fm.embedding[toks[0]], fm.layer_norms[0])
    return d, qb, u


@pytest.mark.parametrize("profile,variant", [("W8A8", "mamba2"), ("W4A8", "mamba2"), ("W4A16", "mamba2"),
                                             ("W8A8", "mamba1"), ("W4A8", "mamba1"), ("W4A16", "mamba1")])
def test_block_forward_quantized(cuda, profile, variant):
    from paper_2503_22879_b200.ssm_block import block_forward_quantized, DeviceBlock
    d, qb, u = _tiny_block(profile, variant)
    tr = {}
    ref, rst = oq.block_forward_quantized(u, qb, trace=tr)
    blk = DeviceBlock(qb, cuda)
    out, st = block_forward_quantized(torch.as_tensor(u, device=cuda), blk)
    out = out.cpu().numpy()
    rel = np.abs(out - ref).max() / np.abs(ref).max()
    assert rel < (2e-2 if qb.a8 else 1e-3), rel
    if qb.a8:
        h = st.h.cpu().numpy().reshape(rst.h.shape)
        mx, frac = code_diff(h, rst.h)
        assert mx <= 1 and frac < 2e-2
        cc = st.conv_cache.cpu().numpy()[0].T
        assert np.array_equal(cc, rst.conv)
    else:   # float state and conv cache
        h = st.h.cpu().numpy().reshape(rst.h.shape)
        assert np.abs(h - rst.h).max() <= 1e-3 * np.abs(rst.h).max() + 1e-6
        cc = st.conv_cache.cpu().numpy()[0].T   # conv inputs = in_proj outputs (GEMV vs BLAS order)
        assert np.abs(cc - rst.conv).max() <= 1e-4 * np.abs(rst.conv).max()


@pytest.mark.parametrize("profile,variant", [("W8A8", "mamba2"), ("W4A8", "mamba2"), ("W4A16", "mamba2"),
                                             ("W8A8", "mamba1"), ("W4A8", "mamba1"), ("W4A16", "mamba1")])
def test_decode_matches_oracle_steps(cuda, profile, variant):
    """Prefill 48 tokens then 16 single-token decode steps (cached state)."""
    from paper_2503_22879_b200.ssm_block import block_forward_quantized, DeviceBlock
    d, qb, u = _tiny_block(profile, variant)
    blk = DeviceBlock(qb, cuda)
    _, ost = oq.block_forward_quantized(u[:48], qb)
    _, gst = block_forward_quantized(torch.as_tensor(u[:48], device=cuda), blk)
    worst = 0.0
    for t in range(48, 64):
        ro, ost = oq.block_forward_quantized(u[t:t + 1], qb, ost)
        go, gst = block_forward_quantized(torch.as_tensor(u[t:t + 1], device=cuda), blk, state=gst)
        worst = max(worst, np.abs(go.cpu().numpy() - ro).max() / np.abs(ro).max())
    assert worst < 5e-2, worst


@pytest.mark.parametrize("M,N,K", [(64, 4096, 8192), (64, 8192, 4096), (16, 1024, 8192), (64, 256000 // 8, 4096)])
def test_gemm_w4a8_tc_repeat_deterministic(cuda, M, N, K):
    """Split-K cluster reduction, persistent multi-unit CTAs and the async rings: 6 launches on
    fresh data, every one bit-exact against the oracle's promotion order."""
    ops = _ops()
    r = _rng(9, M, N)
    splits = ops.gemm_w4a8_splits(M, N, K)
    for _ in range(6):
        a, ql, tw, tws = _w4a8_case(r, M, N, K, 128, cuda)
        got = ops.gemm_w4a8(torch.as_tensor(a, device=cuda), tw, tws, 128, 0.01, N, ops.EPI_F32).cpu().numpy()
        _same(got, oq.qlinear_a8(a, ql, np.float32(0.01), splits=splits)[0], "repeat")


@pytest.fixture(params=[64, 128], ids=["mma_sync", "tcgen05"])
def ssd_mode(request, cuda):
    """The SSD engine is chosen per call by the chunk argument (128 = tcgen05)."""
    return request.param


@pytest.mark.parametrize("B,T,nh,G,N,seed", [(2, 300, 80, 1, 128, 0), (1, 64, 8, 2, 64, 1), (3, 129, 16, 4, 128, 2)])
def test_ssd_chunk_scan_vs_oracle(cuda, ssd_mode, B, T, nh, G, N, seed):
    """Tensor-core chunked SSD (sq_ssd_scan_int8, T > 1) vs the oracle's sequential f32 scan on
    the same int8 codes: y rel-err <= 5e-3, final int8 state within one step (mismatch < 2e-2),
    with and without an incoming state (chunked prefill continuation)."""
    ops = _ops()
    from paper_2503_22879_b200.ssm_block import SsmState  # noqa: F401
    r = _rng(12, seed)
    P = 64
    di, gn = nh * P, G * N
    hg = (np.arange(nh) // (nh // G)).astype(np.int32)
    A = (-np.exp(r.uniform(0, 2.7, nh))).astype(np.float32)
    D = np.ones(nh, np.float32)
    dtb = (np.log(np.expm1(r.uniform(1e-3, 1e-1, nh)))).astype(np.float32)
    s_x = r.uniform(0.005, 0.02, di).astype(np.float32)
    s_B = r.uniform(0.005, 0.02, G).astype(np.float32)
    s_C = r.uniform(0.005, 0.02, G).astype(np.float32)
    s_h = r.uniform(0.002, 0.01, di).astype(np.float32)
    s_dt, s_z = np.float32(0.03), np.float32(0.03)
    xq = r.integers(-128, 128, (B * T, di)).astype(np.int8)
    Bq = r.integers(-128, 128, (B * T, gn)).astype(np.int8)
    Cq = r.integers(-128, 128, (B * T, gn)).astype(np.int8)
    dq = r.integers(-128, 128, (B * T, nh)).astype(np.int8)
    zq = r.integers(-128, 128, (B * T, di)).astype(np.int8)
    h0 = r.integers(-100, 100, (B, nh, P, N)).astype(np.int8)
    t = lambda a: torch.as_tensor(a, device=cuda)
    tens = dict(hg=t(hg), A=t(A), D=t(D), dtb=t(dtb), s_x=t(s_x), s_B=t(s_B), s_C=t(s_C), s_h=t(s_h))
    prm = ops.mamba2_params(nh, P, N, G, tens["hg"], tens["A"], tens["D"], tens["dtb"], s_dt, s_z, tens["s_x"],
                            tens["s_B"], tens["s_C"], tens["s_h"])
    for state_in in (False, True):
        st = t(h0.copy())
        y = torch.empty((B * T, di), dtype=torch.float32, device=cuda)
        ops.ssd_scan_int8(prm, B, T, t(xq), t(Bq), t(Cq), t(dq), t(zq), st, state_in, y, chunk=ssd_mode)
        y = y.cpu().numpy()
        st = st.cpu().numpy()
        for bi in range(B):
            sl = slice(bi * T, (bi + 1) * T)
            x = (xq[sl].astype(np.float32) * s_x).reshape(T, nh, P)
            Bh = (Bq[sl].astype(np.float32).reshape(T, G, N) * s_B[None, :, None]).astype(np.float32)
            Ch = (Cq[sl].astype(np.float32).reshape(T, G, N) * s_C[None, :, None]).astype(np.float32)
            dA, dt = osb.discretize((dq[sl].astype(np.float32) * s_dt).astype(np.float32), dtb, A)
            z = (zq[sl].astype(np.float32) * s_z).reshape(T, nh, P)
            hin = (h0[bi].astype(np.float32) * s_h.reshape(nh, P)[:, :, None]) if state_in else None
            ry, rh = osb.selective_scan(x, dA, dt, Bh, Ch, D, z, hin, hg)
            rel = np.abs(y[sl] - ry.reshape(T, di)).max() / np.abs(ry).max()
            assert rel <= 5e-3, (state_in, bi, rel)
            rq = quantize_codes(rh, s_h.reshape(nh, P)[:, :, None], 8)
            mx, frac = code_diff(st[bi], rq)
            assert mx <= 1 and frac < 2e-2, (state_in, bi, mx, frac)


@pytest.mark.parametrize("B,T,nh,G,N", [(1, 1, 128, 8, 128), (2, 5, 16, 2, 64), (1, 16, 32, 4, 128), (2, 3, 8, 1, 256)])
def test_ssd_scan_f32_vs_oracle(cuda, B, T, nh, G, N):
    """W4A16 float scan (sq_ssd_scan_f32: decode T=1 at the Mamba2-8B head shape, short prompts)
    vs the oracle's sequential f32 selective scan: y rel-err <= 1e-4; the state is the same
    element-wise f32 recurrence (rel <= 1e-5: exp / log1p ulps), with and without an incoming state."""
    ops = _ops()
    r = _rng(13, B * 1000 + T, nh * 1000 + N)
    P = 64
    di, gn = nh * P, G * N
    hg = (np.arange(nh) // (nh // G)).astype(np.int32)
    A = (-np.exp(r.uniform(0, 2.7, nh))).astype(np.float32)
    D = r.uniform(0.5, 1.5, nh).astype(np.float32)
    dtb = (np.log(np.expm1(r.uniform(1e-3, 1e-1, nh)))).astype(np.float32)
    x = r.standard_normal((B * T, di)).astype(np.float32)
    Bm = r.standard_normal((B * T, gn)).astype(np.float32)
    Cm = r.standard_normal((B * T, gn)).astype(np.float32)
    dr = (r.standard_normal((B * T, nh)) * 0.5).astype(np.float32)
    z = r.standard_normal((B * T, di)).astype(np.float32)
    h0 = (r.standard_normal((B, nh, P, N)) * 0.3).astype(np.float32)
    t = lambda a: torch.as_tensor(a, device=cuda)
    tens = dict(hg=t(hg), A=t(A), D=t(D), dtb=t(dtb))
    prm = ops.mamba2_params(nh, P, N, G, tens["hg"], tens["A"], tens["D"], tens["dtb"])
    for state_in in (False, True):
        st = t(h0.copy())
        y = torch.empty((B * T, di), dtype=torch.float32, device=cuda)
        ops.ssd_scan_f32(prm, B, T, t(x), t(Bm), t(Cm), t(dr), t(z), st, state_in, y)
        y, st = y.cpu().numpy(), st.cpu().numpy()
        for bi in range(B):
            sl = slice(bi * T, (bi + 1) * T)
            dA, dt = osb.discretize(dr[sl], dtb, A)
            ry, rh = osb.selective_scan(x[sl].reshape(T, nh, P), dA, dt, Bm[sl].reshape(T, G, N),
                                        Cm[sl].reshape(T, G, N), D, z[sl].reshape(T, nh, P),
                                        h0[bi] if state_in else None, hg)
            rel = np.abs(y[sl] - ry.reshape(T, di)).max() / np.abs(ry).max()
            assert rel <= 1e-4, (state_in, bi, rel)
            hrel = np.abs(st[bi] - rh).max() / np.abs(rh).max()
            assert hrel <= 1e-5, (state_in, bi, hrel)


@pytest.mark.parametrize("B,T,d_inner", [(1, 1024, 128), (2, 700, 64)])
def test_mamba1_scan_time_chunked_matches_single_pass(cuda, B, T, d_inner):
    """The time-chunked two-pass Mamba1 int8 scan (ws given: chunk end states + decay products,
    then the carried start states) equals the single pass (oracle-tested above) up to f32
    rounding of the carried states: y rel <= 1e-5, final state codes within one step."""
    ops = _ops()
    from paper_2503_22879_b200 import synth
    from paper_2503_22879_b200.ssm_block import DeviceBlock, Dims
    d = Dims("mamba1", 64, d_inner, 16, 1, d_inner, 1, 4, dt_rank=8)
    blk = DeviceBlock(synth.random_qblock(d, "W8A8", 4), cuda)
    g = torch.Generator(device=cuda)
    g.manual_seed(B * T)
    x, dt, z = (torch.randint(-100, 100, (B * T, d_inner), dtype=torch.int8, device=cuda, generator=g) for _ in range(3))
    bc = torch.randint(-100, 100, (B * T, 32), dtype=torch.int8, device=cuda, generator=g)
    nb = int(ops.lib().sq_selective_scan_int8_ws_bytes(ops.C.byref(blk.params), B, T))
    assert nb > 0   # this shape takes the chunked path
    h0 = torch.randint(-60, 60, (B, d_inner, 16), dtype=torch.int8, device=cuda, generator=g)
    outs = []
    for chunked in (False, True):
        st = h0.clone()
        y = torch.empty((B * T, d_inner), device=cuda)
        if chunked:
            ops.selective_scan_int8(blk.params, B, T, x, dt, bc, z, st, True, y)
        else:   # single pass: no workspace
            ops._check(ops.lib().sq_selective_scan_int8(ops.C.byref(blk.params), B, T, x.data_ptr(), d_inner,
                                                        dt.data_ptr(), d_inner, bc.data_ptr(), 32, z.data_ptr(),
                                                        d_inner, st.data_ptr(), 1, y.data_ptr(), d_inner, None,
                                                        ops._stream()))
        outs.append((y, st))
    (y1, s1), (y2, s2) = outs
    assert ((y2 - y1).abs().max() / y1.abs().max()).item() <= 1e-5
    assert (s2.int() - s1.int()).abs().max().item() <= 1
