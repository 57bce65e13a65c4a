"""GPU parity of the fused Mamba2 decode step (sq_mamba2_decode_step_int8) against the
oracle's batched decode step (oracle/qblock.py decode_step_batched), on the kernel's
own input codes so each output is checked in isolation:

* conv cache: bit-exact;
* int8 SSM state codes: within one quantization step, mismatch fraction < 1e-3;
* y (pre-norm, f32): rel-err <= 1e-3 (f32 FMA order vs the oracle's f64 sum);
* yq (out_proj input codes after norm + FWHT + quant): within one step, mismatch < 1e-3.
Shapes: tiny (cluster of 2 with a cross-CTA Hadamard stage), Mamba2-2.7B (cluster of 5,
non-power-of-two d_inner), Mamba2-8B (cluster of 8, three cross-CTA stages), with and
without a head permutation (reordered heads -> state groups interleaved).
"""
import numpy as np
import pytest
import torch

from oracle import qblock as oq
from oracle import ssm_block as osb

pytestmark = pytest.mark.gpu

SHAPES = {
    "tiny": (("mamba2", 256, 512, 64, 8, 64, 2, 4), 3),
    "m2_2p7b": (("mamba2", 2560, 5120, 128, 80, 64, 1, 4), 4),
    "m2_8b": (("mamba2", 4096, 8192, 128, 128, 64, 8, 4), 64),
}


def _to_oracle(pqb):
    od = osb.Dims(**vars(pqb.dims))
    return oq.QBlock(od, pqb.profile, oq.QLinear(**vars(pqb.in_proj)), oq.QLinear(**vars(pqb.out_proj)),
                     pqb.conv_weight, pqb.conv_bias, pqb.a_log, pqb.d_param, pqb.dt_bias, pqb.norm_weight,
                     pqb.head_group, s_u=pqb.s_u, in_out_scale=pqb.in_out_scale, conv_in_scale=pqb.conv_in_scale,
                     conv_out_scale=pqb.conv_out_scale, state_scale=pqb.state_scale, s_y=pqb.s_y)


def _diff(a, b):
    d = np.abs(np.asarray(a, np.int32) - np.asarray(b, np.int32))
    return int(d.max(initial=0)), float((d > 0).mean())


@pytest.mark.parametrize("permute", [False, True], ids=["ordered", "reordered"])
@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_fused_decode_step(cuda, shape, permute):
    from paper_2503_22879_b200 import ops, synth
    from paper_2503_22879_b200.ssm_block import DeviceBlock, Dims
    dims, B = SHAPES[shape]
    d = Dims(*dims)
    pqb = synth.random_qblock(d, "W8A8" if shape == "tiny" else "W4A8", seed=5)
    if permute:   # reordered heads: a head permutation moves state groups around
        perm = np.random.default_rng(1).permutation(d.n_heads)
        pqb.head_group = pqb.head_group[perm].astype(np.int32)
    qb = _to_oracle(pqb)
    r = np.random.default_rng(2)
    u = r.standard_normal((B, d.d_model)).astype(np.float32)
    h0 = r.integers(-100, 100, (B, d.n_heads, d.head_dim, d.d_state)).astype(np.int8)
    c0 = r.integers(-100, 100, (B, d.conv_dim, d.conv_kernel - 1)).astype(np.int8)
    tr = {}
    _, rh, rc = oq.decode_step_batched(u, qb, h0, c0, trace=tr)
    blk = DeviceBlock(pqb, cuda)
    assert blk.fused_decode
    zx = torch.as_tensor(tr["in_codes"], device=cuda)
    st = torch.as_tensor(h0, device=cuda)
    cc = torch.as_tensor(np.ascontiguousarray(c0.transpose(0, 2, 1)), device=cuda)
    y = torch.empty((B, d.d_inner), dtype=torch.float32, device=cuda)
    gs = torch.zeros((B, d.d_inner // 128), dtype=torch.int32, device=cuda)
    yq = ops.mamba2_decode_step_int8(blk.decode_params, B, zx, cc, st, y=y, gsum=gs)
    torch.cuda.synchronize()
    assert np.array_equal(gs.cpu().numpy(), yq.cpu().numpy().astype(np.int32).reshape(B, -1, 128).sum(-1))
    assert np.array_equal(cc.cpu().numpy().transpose(0, 2, 1), rc), "conv cache must be bit-exact"
    mx, frac = _diff(st.cpu().numpy(), rh)
    assert mx <= 1 and frac < 1e-3, (mx, frac)
    yr = tr["y"]
    rel = np.abs(y.cpu().numpy() - yr).max() / np.abs(yr).max()
    # y = C·h over N = 128 state columns: f32 FMA chains in the kernel vs the oracle's f64 einsum
    # (codes at full int8 range make |h| large against |y|); the contract is on the codes below
    assert rel <= 1e-3, rel
    mx, frac = _diff(yq.cpu().numpy(), tr["y_q"])
    assert mx <= 1 and frac < 1e-3, (mx, frac)


def test_fused_decode_repeat_deterministic(cuda):
    """Cluster reductions run in fixed rank order: repeated launches are bit-identical."""
    from paper_2503_22879_b200 import ops, synth
    from paper_2503_22879_b200.ssm_block import Dims
    d = Dims(*SHAPES["m2_8b"][0])
    blk = synth.device_qblock(d, "W4A8", 0, cuda)
    B = 16
    zx = torch.randint(-128, 128, (B, d.in_proj_out), dtype=torch.int8, device=cuda)
    h = torch.randint(-100, 100, (B, d.n_heads, d.head_dim, d.d_state), dtype=torch.int8, device=cuda)
    cc = torch.randint(-100, 100, (B, 3, d.conv_dim), dtype=torch.int8, device=cuda)
    outs = []
    for _ in range(3):
        h1, c1 = h.clone(), cc.clone()
        yq = ops.mamba2_decode_step_int8(blk.decode_params, B, zx, c1, h1)
        outs.append((yq.cpu(), h1.cpu(), c1.cpu()))
    for o in outs[1:]:
        for a, b in zip(o, outs[0]):
            assert torch.equal(a, b)


M1_SHAPES = {
    "tiny": (("mamba1", 256, 512, 16, 1, 512, 1, 4, 32), 3),
    "m1_2p8b": (("mamba1", 2560, 5120, 16, 1, 5120, 1, 4, 160), 1),
    "m1_2p8b_b8": (("mamba1", 2560, 5120, 16, 1, 5120, 1, 4, 160), 8),
}


@pytest.mark.parametrize("shape", sorted(M1_SHAPES))
def test_mamba1_fused_decode_matches_launch_chain(cuda, shape):
    """The one-launch Mamba1 W8A8 decode step (sq_mamba1_decode_step_int8: conv update, x_proj,
    dt_proj, scan step, gated norm + FWHT + quant behind grid barriers) against the five-launch
    chain it replaces (sq_conv1d_update_int8, two tcgen05 W8A8 GEMMs, the T=1 scan kernel,
    sq_gate_norm_had_quant), three steps in a row on the same codes: conv cache and int8 state
    bit-exact, yq within one step (Σy² is summed in another fixed order), mismatch < 1e-3."""
    from paper_2503_22879_b200 import ops, synth
    from paper_2503_22879_b200.ssm_block import EPS_NORM, DeviceBlock, Dims
    dims, B = M1_SHAPES[shape]
    d = Dims(*dims)
    blk = DeviceBlock(synth.random_qblock(d, "W8A8", seed=7), cuda)
    assert blk.m1_fused_decode
    di, R = d.d_inner, d.dt_rank
    g = torch.Generator(device=cuda)
    g.manual_seed(11)
    h0 = torch.randint(-100, 100, (B, 1, di, 16), dtype=torch.int8, device=cuda, generator=g)
    c0 = torch.randint(-100, 100, (B, d.conv_kernel - 1, di), dtype=torch.int8, device=cuda, generator=g)
    hf, cf, hu, cu = h0.clone(), c0.clone(), h0.clone(), c0.clone()
    ws = torch.zeros(ops.mamba1_decode_ws_bytes(blk.m1_decode_params, B), dtype=torch.uint8, device=cuda)
    for step in range(3):
        zx = torch.randint(-128, 128, (B, 2 * di), dtype=torch.int8, device=cuda, generator=g)
        yf = ops.mamba1_decode_step_int8(blk.m1_decode_params, B, zx, cf, hf, ws)
        cv = ops.conv1d_update_int8(zx[:, di:], blk.conv_w, blk.conv_b, blk.conv_in_scale, blk.conv_out_scale, cu)
        xd = blk.x_proj.a8(cv, ops.EPI_QUANT, None, blk.xproj_out_scale)
        dtq = blk.dt_proj.a8(xd[:, :R].contiguous(), ops.EPI_QUANT, None, blk.dt_scale)
        y = torch.empty((B, di), device=cuda)
        ops.selective_scan_int8(blk.params, B, 1, cv, dtq, xd[:, R:], zx[:, :di], hu, True, y)
        yu = ops.gate_norm_had_quant(y, blk.norm_w, EPS_NORM, blk.s_y, blk.hadamard)
        torch.cuda.synchronize()
        assert torch.equal(cf, cu), step
        assert torch.equal(hf, hu), step
        mx, frac = _diff(yf.cpu().numpy(), yu.cpu().numpy())
        assert mx <= 1 and frac < 1e-3, (step, mx, frac)


def test_mamba1_fused_decode_repeat_deterministic(cuda):
    """The grid-barrier counters reset themselves: repeated launches on one workspace agree bit
    for bit."""
    from paper_2503_22879_b200 import ops, synth
    from paper_2503_22879_b200.ssm_block import DeviceBlock, Dims
    d = Dims(*M1_SHAPES["m1_2p8b"][0])
    blk = DeviceBlock(synth.random_qblock(d, "W8A8", seed=3), cuda)
    B = 2
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    zx = torch.randint(-128, 128, (B, 2 * d.d_inner), dtype=torch.int8, device=cuda, generator=g)
    h = torch.randint(-100, 100, (B, 1, d.d_inner, 16), dtype=torch.int8, device=cuda, generator=g)
    cc = torch.randint(-100, 100, (B, 3, d.d_inner), dtype=torch.int8, device=cuda, generator=g)
    ws = torch.zeros(ops.mamba1_decode_ws_bytes(blk.m1_decode_params, B), dtype=torch.uint8, device=cuda)
    outs = []
    for _ in range(4):
        h1, c1 = h.clone(), cc.clone()
        yq = ops.mamba1_decode_step_int8(blk.m1_decode_params, B, zx, c1, h1, ws)
        outs.append((yq.cpu(), h1.cpu(), c1.cpu()))
    for o in outs[1:]:
        for a, b in zip(o, outs[0]):
            assert torch.equal(a, b)


@pytest.mark.parametrize("dims,B", [(("mamba1", 256, 512, 16, 1, 512, 1, 4, 32), 2),
                                    (("mamba1", 2560, 5120, 16, 1, 5120, 1, 4, 160), 1)], ids=["tiny", "m1_2p8b"])
def test_mamba1_decode_layer_in_one_launch(cuda, dims, B):
    """Whole-layer Mamba1 W8A8 decode (sq_mamba1_decode_layer_int8: pre-norm + quant in the
    rmsnorm16 summation order, in_proj, the SSM half, out_proj residual) equals the four-launch
    chain per decode step: residual stream, conv caches and int8 states bit-exact over 4 steps
    of a 3-layer model; the CUDA-graph generate agrees token for token."""
    from paper_2503_22879_b200 import ops, synth
    from paper_2503_22879_b200.ssm_block import Dims
    d = Dims(*dims)
    m = synth.synthetic_lm(d, 3, "W8A8", 512, cuda, seed=4, head_kind="w8")
    assert all(b.m1_fused_decode for b in m.blocks)
    g = torch.Generator(device=cuda)
    g.manual_seed(8)
    prompt = torch.randint(0, 512, (B, 12), generator=g, device=cuda)
    _, st0 = m.prefill(prompt)
    runs = []
    for fuse in (True, False):
        m.fuse_layers = fuse
        sts = [type(s)(s.h.clone(), s.conv_cache.clone()) for s in st0]
        ws = m._workspace(B)
        tok = torch.empty(B, dtype=torch.int32, device=cuda)
        tok.copy_(prompt[:, -1])
        lgs = []
        for _ in range(4):
            lg = m.decode_step(tok, sts, ws)
            lgs.append(lg.clone())
            tok = ops.argmax(lg)
        torch.cuda.synchronize()
        runs.append((lgs, sts))
    (lf, sf), (lu, su) = runs
    for a, b in zip(lf, lu):
        assert torch.equal(a, b)
    for a, b in zip(sf, su):
        assert torch.equal(a.h, b.h) and torch.equal(a.conv_cache, b.conv_cache)
    m.fuse_layers = True
    out_f = m.generate(prompt, 6)
    m.fuse_layers = False
    out_u = m.generate(prompt, 6)
    assert torch.equal(out_f, out_u)
    assert not synth.synthetic_lm(d, 1, "W8A8", 512, cuda, seed=5, head_kind="w8").fuse_layers   # default off
