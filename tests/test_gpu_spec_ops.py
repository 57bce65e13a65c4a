"""GPU parity of the SPEC float ops exported by ssmquant.ssm_block against
the oracle restatement (oracle/ssm_block.py), on the same seeded inputs:

* project_inputs: slices of one float GEMM, rel <= 1e-6 (f64 accumulation on both sides);
* causal_conv1d: rel <= 1e-6; cache stepping == full sequence;
* discretize: SPEC examples (Δ = ln 2 → Ȧ = 0.5) and rel <= 1e-6;
* selective_scan (Mamba2 and Mamba1 forms, SPEC scalar example h₁ = ln 2): rel <= 1e-5;
* ssd_chunked: == selective_scan for every chunk, <= 1e-4 vs the oracle's chunked SSD;
* block_forward_float: rel <= 1e-4 of the oracle, and token-by-token stepping with the
  returned SsmState equals the full-sequence forward <= 1e-5.
"""
import numpy as np
import pytest
import torch

from oracle import ssm_block as osb
from oracle.tensor_core import make_rng

pytestmark = pytest.mark.gpu


def _sb():
    from paper_2503_22879_b200 import ssm_block
    return ssm_block


def _rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def _toy(variant, seed=0):
    from oracle import pipeline as opl
    if variant == "mamba2":
        d = osb.Dims("mamba2", 64, 128, 16, 8, 16, 2, 4)     # SPEC.md:354 toy dims
    else:
        d = osb.Dims("mamba1", 64, 128, 16, 1, 128, 1, 4, dt_rank=8)
    fm = opl.cmd_gen_toy(d, 1, seed=seed, vocab=64)
    return d, fm.blocks[0]


def _weights(w):
    from paper_2503_22879_b200.ssm_block import Dims, SsmBlockWeights
    d = Dims(**vars(w.dims))
    return SsmBlockWeights(d, w.in_proj, w.conv_weight, w.conv_bias, w.a_log, w.d_param, w.dt_bias, w.norm_weight,
                           w.out_proj, w.x_proj, w.dt_proj, w.head_group)


@pytest.mark.parametrize("variant", ["mamba2", "mamba1"])
def test_project_inputs(cuda, variant):
    sb = _sb()
    d, w = _toy(variant)
    u = make_rng(3, 1).standard_normal((37, d.d_model)).astype(np.float32)
    got = sb.project_inputs(torch.as_tensor(u, device=cuda), _weights(w))
    ref = osb.project_inputs(u, w)
    for g, r in zip(got, ref):
        assert (g is None) == (r is None)
        if r is not None:
            assert _rel(g, r) <= 1e-6


def test_causal_conv1d_and_cache_stepping(cuda):
    sb = _sb()
    r = make_rng(3, 2)
    T, C, K = 50, 96, 4
    x = r.standard_normal((T, C)).astype(np.float32)
    w = (r.standard_normal((C, K)) * 0.5).astype(np.float32)
    b = (r.standard_normal(C) * 0.1).astype(np.float32)
    cache = r.standard_normal((C, K - 1)).astype(np.float32)
    tx = torch.as_tensor(x, device=cuda)
    ry, rc = osb.causal_conv1d(x, w, b, cache)
    gy, gc = sb.causal_conv1d(tx, w, b, torch.as_tensor(cache, device=cuda))
    assert _rel(gy, ry) <= 1e-6 and np.array_equal(gc.cpu().numpy(), rc)
    # token-by-token stepping with the cache == the full sequence
    full, _ = sb.causal_conv1d(tx, w, b)
    c = None
    steps = []
    for t in range(T):
        yt, c = sb.causal_conv1d(tx[t:t + 1], w, b, c)
        steps.append(yt)
    assert _rel(torch.cat(steps), full.cpu().numpy()) <= 1e-6
    # kernel=1, weight=1, bias=0 -> SiLU(x)
    y1, _ = sb.causal_conv1d(tx, np.ones((C, 1), np.float32), np.zeros(C, np.float32))
    assert _rel(y1, osb.silu(x)) <= 1e-6


def test_discretize(cuda):
    sb = _sb()
    ln2 = np.float32(np.log(2.0))
    # A=-1, Δ_raw + bias with Δ = ln 2 -> Ȧ = 0.5; Δ_raw = dt_bias = 0 -> Δ = ln 2
    raw = np.array([[np.log(np.expm1(ln2)), 0.0]], np.float32)
    dA, dt = sb.discretize(torch.as_tensor(raw, device=cuda), np.zeros(2, np.float32), np.array([-1.0, -1.0], np.float32))
    assert abs(dA.cpu().numpy()[0, 0] - 0.5) <= 1e-6 and abs(dt.cpu().numpy()[0, 1] - ln2) <= 1e-6
    r = make_rng(3, 3)
    raw = (r.standard_normal((20, 12)) * 3).astype(np.float32)
    bias = r.standard_normal(12).astype(np.float32)
    for A in (-np.exp(r.standard_normal(12)).astype(np.float32), -np.exp(r.standard_normal((12, 16))).astype(np.float32)):
        gA, gd = sb.discretize(torch.as_tensor(raw, device=cuda), bias, A)
        rA, rd = osb.discretize(raw, bias, A)
        assert _rel(gA, rA) <= 1e-6 and _rel(gd, rd) <= 1e-6


def test_selective_scan_spec_scalar(cuda):
    """A=-1, Δ=ln2, B=C=1, D=0, x=[1], h0=0 -> h1 = ln 2 (pre-gating y1 = ln 2), Mamba1 form."""
    sb = _sb()
    ln2 = np.float32(np.log(2.0))
    t = lambda a: torch.as_tensor(np.asarray(a, np.float32), device=cuda)   # noqa: E731
    dA = np.full((1, 1, 16), 0.5, np.float32)
    Bm = np.zeros((1, 16), np.float32)
    Bm[0, 0] = 1
    y, h = sb.selective_scan(t([[1.0]]), t(dA), t([[ln2]]), t(Bm), t(Bm), np.zeros(1, np.float32))
    assert abs(h.cpu().numpy()[0, 0, 0] - ln2) <= 1e-6 and abs(y.cpu().numpy()[0, 0] - ln2) <= 1e-6


@pytest.mark.parametrize("with_state", [False, True])
def test_selective_scan_and_ssd_chunked(cuda, with_state):
    sb = _sb()
    r = make_rng(3, 4, int(with_state))
    T, nh, P, G, N = 45, 8, 32, 2, 64
    x = r.standard_normal((T, nh, P)).astype(np.float32)
    dA = np.exp(-np.abs(r.standard_normal((T, nh))) * 0.3).astype(np.float32)
    dt = np.abs(r.standard_normal((T, nh)) * 0.2).astype(np.float32)
    Bm = r.standard_normal((T, G, N)).astype(np.float32)
    Cm = r.standard_normal((T, G, N)).astype(np.float32)
    D = r.standard_normal(nh).astype(np.float32)
    z = r.standard_normal((T, nh, P)).astype(np.float32)
    h0 = r.standard_normal((nh, P, N)).astype(np.float32) if with_state else None
    hg = np.array([1, 0, 1, 0, 0, 1, 1, 0], np.int32)              # permuted heads (reordered model)
    t = lambda a: None if a is None else torch.as_tensor(a, device=cuda)   # noqa: E731
    ry, rh = osb.selective_scan(x, dA, dt, Bm, Cm, D, z, h0, hg)
    gy, gh = sb.selective_scan(t(x), t(dA), t(dt), t(Bm), t(Cm), D, t(z), t(h0), hg)
    assert _rel(gy, ry) <= 1e-5 and _rel(gh, rh) <= 1e-5
    gy0, _ = sb.selective_scan(t(x), t(dA), t(dt), t(Bm), t(Cm), D, None, t(h0), hg)   # ungated
    ry0, _ = osb.selective_scan(x, dA, dt, Bm, Cm, D, None, h0, hg)
    assert _rel(gy0, ry0) <= 1e-5
    for chunk in (1, 3, 16, T):
        cy, ch = sb.ssd_chunked(t(x), t(dA), t(dt), t(Bm), t(Cm), D, t(z), chunk, t(h0), hg)
        oy, oh = osb.ssd_chunked(x, dA, dt, Bm, Cm, D, z, chunk, h0, hg)
        assert _rel(cy, oy) <= 1e-4 and _rel(ch, oh) <= 1e-4
    # Mamba1 form
    d = 48
    x1 = r.standard_normal((T, d)).astype(np.float32)
    dA1 = np.exp(-np.abs(r.standard_normal((T, d, 16))) * 0.3).astype(np.float32)
    dt1 = np.abs(r.standard_normal((T, d)) * 0.2).astype(np.float32)
    B1, C1 = r.standard_normal((T, 16)).astype(np.float32), r.standard_normal((T, 16)).astype(np.float32)
    z1, D1 = r.standard_normal((T, d)).astype(np.float32), r.standard_normal(d).astype(np.float32)
    s1 = r.standard_normal((1, d, 16)).astype(np.float32) if with_state else None
    ry, rh = osb.selective_scan(x1, dA1, dt1, B1, C1, D1, z1, s1)
    gy, gh = sb.selective_scan(t(x1), t(dA1), t(dt1), t(B1), t(C1), D1, t(z1), t(s1))
    assert _rel(gy, ry) <= 1e-5 and _rel(gh, rh) <= 1e-5


@pytest.mark.parametrize("variant", ["mamba2", "mamba1"])
def test_block_forward_float(cuda, variant):
    sb = _sb()
    d, w = _toy(variant, seed=2)
    pw = _weights(w)
    u = make_rng(3, 5).standard_normal((24, d.d_model)).astype(np.float32)
    ro, rs = osb.block_forward_float(u, w)
    tu = torch.as_tensor(u, device=cuda)
    go, gs = sb.block_forward_float(tu, pw)
    assert _rel(go, ro) <= 1e-4
    assert _rel(gs.h, rs.h) <= 1e-4 and _rel(gs.conv_cache, rs.conv_cache) <= 1e-6
    if variant == "mamba2":
        gc, _ = sb.block_forward_float(tu, pw, chunk=8)
        assert _rel(gc, go.cpu().numpy()) <= 1e-5
    # stateful single-token stepping == full-sequence forward
    st = None
    outs = []
    for t in range(u.shape[0]):
        o, st = sb.block_forward_float(tu[t:t + 1], pw, st)
        outs.append(o)
    assert _rel(torch.cat(outs), go.cpu().numpy()) <= 1e-5
