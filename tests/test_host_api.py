"""CPU: the product's host-side (offline) API against the test oracle — SURVEY §8 a13-a15.

Weight codes, u4 packing, ClusterMaps, reorder permutations and every scale table must be
bit-exact (north_star); the float calibration forward (torch) agrees with the oracle's
within float tolerance, and fed the same statistics the whole quantize pipeline produces
identical quantized models.
"""
import numpy as np
from paper_2503_22879_b200.errors import CalibrationError
import pytest
import torch

from oracle import calibrate as ocal
from oracle import hadamard as ohad
from oracle import pipeline as opl
from oracle import quantizer as oqz
from oracle import reorder as oro
from oracle import tensor_core as otc
from oracle.ssm_block import Dims as ODims
from paper_2503_22879_b200 import archive, calibrate, cli, hadamard, quantizer, reorder
from paper_2503_22879_b200.ssm_block import Dims

TINY2 = ("mamba2", 64, 128, 16, 8, 16, 2, 4)
TINY1 = ("mamba1", 64, 128, 16, 1, 128, 1, 4, 8)


def _np(t):
    return t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def test_weight_quantizers_bit_exact():
    r = otc.make_rng(31)
    w = (r.standard_normal((24, 256)) * np.exp(r.uniform(-3, 3, (1, 256)))).astype(np.float32)
    w[3, :128] = 0.0                                        # a zero group -> scale 1.0
    a, b = oqz.quantize_weight_w8(w), quantizer.quantize_weight_w8(w)
    assert np.array_equal(a.payload, _np(b.payload)) and np.array_equal(a.extra["s_ch"], _np(b.extra["s_ch"]))
    a, b = oqz.quantize_weight_w4_group(w, 128), quantizer.quantize_weight_w4(w, 128)
    assert np.array_equal(a.payload, _np(b.payload)) and np.array_equal(a.extra["s_group"], _np(b.extra["s_group"]))
    a, b = oqz.quantize_weight_w4a8(w, 128), quantizer.quantize_weight_w4a8(w, 128)
    assert np.array_equal(a.payload, _np(b.payload)) and np.array_equal(a.extra["s_group"], _np(b.extra["s_group"]))


def test_quantize_layouts_and_spec_examples():
    x = np.array([2.54, -1.27, 0.0], np.float32)
    assert np.isclose(quantizer.compute_scale(x, 8), 0.02)
    assert _np(quantizer.quantize(x, quantizer.ScaleLayout("PerTensor", np.float32(0.02)), 8).payload).tolist() == \
        [127, -64, 0]
    r = otc.make_rng(32)
    v = r.standard_normal((6, 40)).astype(np.float32)
    s = r.uniform(0.01, 0.1, 5).astype(np.float32)
    for lay_o, lay_p in [
        (oqz.ScaleLayout("PerGroup", s, axis=1, group_size=8), quantizer.ScaleLayout("PerGroup", s, axis=1, group_size=8)),
        (oqz.ScaleLayout("PerStateGroup", s, axis=1, bounds=(0, 8, 16, 24, 32, 40)),
         quantizer.ScaleLayout("PerStateGroup", s, axis=1, bounds=(0, 8, 16, 24, 32, 40))),
    ]:
        assert np.array_equal(oqz.quantize(v, lay_o, 8).payload, _np(quantizer.quantize(v, lay_p, 8).payload))
    assert quantizer.fuse_scales(0.02, 1.0, 0.04) == np.float32(0.5)


def test_hadamard_bit_exact():
    r = otc.make_rng(33)
    v = r.standard_normal((3, 5120)).astype(np.float32)
    assert np.array_equal(ohad.fwht_blocked(v), _np(hadamard.fwht_blocked(v)))
    v = r.standard_normal((2, 64)).astype(np.float32)
    assert np.array_equal(ohad.fwht(v, ohad.HadamardPlan(64)), _np(hadamard.fwht(v, hadamard.HadamardPlan(64))))
    w = r.standard_normal((16, 40)).astype(np.float32)
    assert np.array_equal(ohad.fuse_hadamard_out_proj(w, 40, 1), _np(hadamard.fuse_hadamard_out_proj(w, 40, 1)))
    assert np.array_equal(ohad.fuse_hadamard_in_proj(w), _np(hadamard.fuse_hadamard_in_proj(w)))
    y = r.standard_normal((4, 128)).astype(np.float32)
    assert np.array_equal(ohad.hadamard_quantize(y, ohad.HadamardPlan(128, "none", 0.3), 8),
                          _np(hadamard.hadamard_quantize(y, hadamard.HadamardPlan(128, "none", 0.3), 8)))


@pytest.mark.parametrize("seed", range(6))
def test_sort_and_cluster_bit_exact(seed):
    r = otc.make_rng(34, seed)
    nh, P = [(8, 16), (16, 64), (4, 8), (80, 64), (128, 64), (1, 512)][seed]
    mx = (np.exp(r.uniform(-3, 3, (nh, P))) * np.exp(r.uniform(-2, 2, (nh, 1)))).astype(np.float32)
    a = ocal.sort_and_cluster(ocal.CalibStats(mx.reshape(-1), 1), nh, P, 4, 4, seed)
    b = calibrate.sort_and_cluster(calibrate.CalibStats(mx.reshape(-1), 1), nh, P, 4, 4, seed)
    for f in ("head_perm", "channel_perm", "head_group_bounds", "channel_group_bounds", "scales"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(a.cell_of_new(), b.cell_of_new())
    X = r.standard_normal((30, 5))
    assert np.array_equal(ocal.kmeans(X, 4, seed), calibrate.kmeans(X, 4, seed))


def test_state_group_scales_and_reorder_bit_exact():
    r = otc.make_rng(35)
    nh, P, G, N = 8, 16, 2, 16
    mx = np.exp(r.uniform(-3, 3, nh * P)).astype(np.float32)
    sb = np.exp(r.uniform(-3, 3, G * N)).astype(np.float32)
    hh = np.exp(r.uniform(-2, 2, nh * P)).astype(np.float32)
    ocm = ocal.sort_and_cluster(ocal.CalibStats(mx, 1), nh, P)
    pcm = calibrate.sort_and_cluster(calibrate.CalibStats(mx, 1), nh, P)
    a = ocal.build_state_group_scales(ocal.CalibStats(sb, 1), ocal.CalibStats(sb * 2, 1), G, N, ocal.CalibStats(hh, 1), ocm)
    b = calibrate.build_state_group_scales(calibrate.CalibStats(sb, 1), calibrate.CalibStats(sb * 2, 1), G, N,
                                           calibrate.CalibStats(hh, 1), pcm)
    for f in ("boundaries", "scales_B", "scales_C", "scales_state"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    d = Dims(*TINY2)
    ob = opl.gen_block(ODims(*TINY2), 3, 0)
    pb = cli.gen_block(d, 3, 0)
    opl_plan = oro.build_reorder_plan(ocm, ob.dims)
    p_plan = reorder.build_reorder_plan(pcm, d)
    assert np.array_equal(opl_plan.pi, p_plan.pi)
    o2, p2 = oro.apply_reorder(ob, opl_plan), reorder.apply_reorder(pb, p_plan)
    for f in ("in_proj", "conv_weight", "conv_bias", "a_log", "d_param", "dt_bias", "norm_weight", "out_proj",
              "head_group"):
        assert np.array_equal(getattr(o2, f), getattr(p2, f)), f
    with pytest.raises(Exception):
        reorder.apply_reorder(p2, p_plan)


@pytest.mark.parametrize("dims", [TINY2, TINY1], ids=["mamba2", "mamba1"])
def test_gen_toy_and_calibration(dims):
    od, d = ODims(*dims), Dims(*dims)
    fo, fp = opl.cmd_gen_toy(od, 2, seed=4, vocab=64), cli.cmd_gen_toy(d, 2, seed=4, vocab=64)
    assert np.array_equal(fo.embedding, fp.embedding) and np.array_equal(fo.head, fp.head)
    for a, b in zip(fo.blocks, fp.blocks):
        for f in ("in_proj", "conv_weight", "a_log", "dt_bias", "out_proj", "x_proj", "dt_proj"):
            assert np.array_equal(getattr(a, f), getattr(b, f)) if getattr(a, f) is not None else getattr(b, f) is None
    toks = opl.calib_tokens(64, 2, 24)
    so = opl.collect_stats(fo, toks)
    sp = calibrate.collect_stats(fp, toks, device="cpu")          # torch float forward
    for lo, lp in zip(so, sp):
        assert lo.keys() == lp.keys()
        for k in lo:
            a, b = lo[k].channel_max, lp[k].channel_max
            assert np.allclose(a, b, rtol=2e-4, atol=1e-6 * np.abs(a).max()), k
    # SPEC.md:384 sites argument: only the requested taps are kept, with the same statistics
    sub = calibrate.collect_stats(fp, toks, sites=["x", "h", "head_in"], device="cpu")
    assert [set(s) for s in sub] == [{"x", "h"}] * len(fp.blocks) + [{"head_in"}]
    for full, part in zip(sp, sub):
        for k in part:
            assert np.array_equal(full[k].channel_max, part[k].channel_max)
    with pytest.raises(CalibrationError):
        calibrate.collect_stats(fp, toks, sites=["nope"], device="cpu")


@pytest.mark.parametrize("profile", ["W8A8", "W4A8", "W4A16"])
@pytest.mark.parametrize("dims", [TINY2, TINY1], ids=["mamba2", "mamba1"])
def test_quantize_pipeline_bit_exact(profile, dims):
    """Same float model + same calibration statistics -> identical quantized model."""
    od, d = ODims(*dims), Dims(*dims)
    fo, fp = opl.cmd_gen_toy(od, 2, seed=5, vocab=64), cli.cmd_gen_toy(d, 2, seed=5, vocab=64)
    toks = opl.calib_tokens(64, 2, 24)
    stats = opl.collect_stats(fo, toks)
    pstats = [{k: calibrate.CalibStats(v.channel_max, v.sample_count, v.values) for k, v in s.items()}
              for s in stats]
    qo = opl.cmd_quantize(fo, toks, profile)
    qp = cli.cmd_quantize(fp, toks, profile, stats=pstats)
    assert np.array_equal(qo.emb_codes, qp.emb_codes) and np.array_equal(qo.emb_scale, qp.emb_scale)
    assert qo.s_head == qp.s_head and np.array_equal(qo.head.codes, qp.head.codes)
    for a, b in zip(qo.blocks, qp.blocks):
        for lin in ("in_proj", "out_proj", "x_proj", "dt_proj"):
            la, lb = getattr(a, lin), getattr(b, lin)
            if la is None:
                assert lb is None
                continue
            for f in ("codes", "s_ch", "s_group"):
                fa, fb = getattr(la, f), getattr(lb, f)
                assert (fa is None and fb is None) or np.array_equal(np.asarray(fa), np.asarray(fb)), (lin, f)
        for f in ("s_u", "s_y", "s_dt", "in_out_scale", "conv_in_scale", "conv_out_scale", "state_scale",
                  "xproj_out_scale", "head_group", "conv_weight", "norm_weight"):
            fa, fb = getattr(a, f), getattr(b, f)
            assert (fa is None and fb is None) or np.array_equal(np.asarray(fa), np.asarray(fb)), f


def test_archive_roundtrip_and_cli(tmp_path):
    p = str(tmp_path / "a.bin")
    archive.archive_write({"w": np.ones((2, 2), np.float32), "q": ("u4packed", np.array([3, -2, -8, 7])),
                           "m": {"x": 1}}, p)
    back = archive.archive_read(p)
    assert back["q"].tolist() == [3, -2, -8, 7] and back["m"] == {"x": 1}
    assert np.array_equal(archive.pack_u4([3, -2]), otc.pack_u4([3, -2]))               # 0xE3
    fm_path, q_path = str(tmp_path / "toy.bin"), str(tmp_path / "q.bin")
    assert cli.main(["gen-toy", "--dims", "mamba2,64,128,16,8,16,2,4", "--blocks", "1", "--vocab", "64",
                     "--out", fm_path]) == 0
    fm = archive.read_float_model(fm_path)
    ref = cli.cmd_gen_toy(Dims(*TINY2), 1, 0, 64)
    assert np.array_equal(fm.blocks[0].in_proj, ref.blocks[0].in_proj)
    assert cli.main(["quantize", "--model", fm_path, "--profile", "W4A8", "--samples", "1", "--seq-len", "8",
                     "--out", q_path]) == 0
    info = archive.inspect(q_path)
    assert info["blocks.0.in_proj.codes"][-1] == "int8" and "blocks.0.state_scale" in info
    assert cli.main(["quantize", "--model", str(tmp_path / "missing.bin"), "--out", q_path]) == 1


@pytest.mark.parametrize("emb_bits", [8, 4])
@pytest.mark.parametrize("profile,dims", [("W4A8", TINY2), ("W8A8", TINY1), ("W4A16", TINY2)],
                         ids=["w4a8-mamba2", "w8a8-mamba1", "w4a16-mamba2"])
def test_quant_archive_roundtrip(tmp_path, profile, dims, emb_bits):
    """write_quant_model -> read_quant_model restores every code, scale table and scalar bit for bit
    (SPEC.md:49-57, 591), including a 4-bit (u4packed) embedding."""
    fm = cli.cmd_gen_toy(Dims(*dims), 2, seed=7, vocab=64)
    toks = opl.calib_tokens(64, 1, 16)
    qm = cli.cmd_quantize(fm, toks, profile, device="cpu", emb_bits=emb_bits)
    if emb_bits == 4:
        assert qm.emb_codes.min() >= -8 and qm.emb_codes.max() <= 7
    p = str(tmp_path / "q.bin")
    archive.write_quant_model(qm, p)
    if emb_bits == 4:
        assert archive.archive_read(p)["emb_codes"].dtype == np.int8
        assert "u4packed" in open(p, "rb").read(4096).decode("utf-8", "ignore")
    back = archive.read_quant_model(p)
    assert back.profiles == qm.profiles and back.extra["emb_bits"] == emb_bits and back.s_head == qm.s_head
    assert np.array_equal(back.emb_codes, qm.emb_codes) and np.array_equal(back.emb_scale, qm.emb_scale)
    for a, b in zip([qm.head] + [getattr(x, f) for x in qm.blocks for f in ("in_proj", "out_proj", "x_proj", "dt_proj")],
                    [back.head] + [getattr(x, f) for x in back.blocks for f in ("in_proj", "out_proj", "x_proj", "dt_proj")]):
        if a is None:
            assert b is None
            continue
        assert a.kind == b.kind and a.group == b.group and np.array_equal(a.codes, b.codes)
        for f in ("s_ch", "s_group"):
            assert (getattr(a, f) is None) == (getattr(b, f) is None)
            if getattr(a, f) is not None:
                assert np.array_equal(np.asarray(getattr(a, f)), getattr(b, f))
    for x, y in zip(qm.blocks, back.blocks):
        for f in ("conv_weight", "conv_bias", "a_log", "d_param", "dt_bias", "norm_weight", "in_out_scale",
                  "conv_in_scale", "conv_out_scale", "state_scale", "xproj_out_scale", "head_group"):
            fa, fb = getattr(x, f), getattr(y, f)
            assert (fa is None) == (fb is None) and (fa is None or np.array_equal(np.asarray(fa), np.asarray(fb))), f
        assert (x.s_u, x.s_y, x.s_dt, x.hadamard, x.profile) == (y.s_u, y.s_y, y.s_dt, y.hadamard, y.profile)


# ---------------------------------------------------------------- oracle-independent properties
# The bit-exact comparisons above check the product against the numpy restatement.  These check
# the product's host transforms against the MATH they must satisfy, so a shared misreading of
# SPEC in both restatements would still fail here.

def _as_oracle_weights(w):
    from oracle import ssm_block as osb
    fields = {f: getattr(w, f) for f in osb.SsmBlockWeights.__dataclass_fields__ if hasattr(w, f)}
    fields["dims"] = osb.Dims(**vars(w.dims))
    return osb.SsmBlockWeights(**fields)


@pytest.mark.parametrize("dims", [TINY2, TINY1], ids=["mamba2", "mamba1"])
def test_reorder_preserves_the_block_function(dims):
    """reordering is a relabelling of the block's channels (and heads), so the
    float block maps the same input to the same output and the final state is the permuted one
    (permute_state)."""
    from oracle import ssm_block as osb
    d = Dims(*dims)
    w = cli.gen_block(d, 5, 0)
    nh, P = (1, d.d_inner) if d.variant == "mamba1" else (d.n_heads, d.head_dim)
    r = np.random.default_rng(4)
    cm = calibrate.sort_and_cluster(calibrate.CalibStats(np.exp(r.uniform(-3, 3, nh * P)).astype(np.float32), 1),
                                    nh, P)
    plan = reorder.build_reorder_plan(cm, d)
    assert not np.array_equal(plan.pi, np.arange(d.d_inner))   # a real permutation
    w2 = reorder.apply_reorder(w, plan)
    u = r.standard_normal((24, d.d_model)).astype(np.float32)
    y1, s1 = osb.block_forward_float(u, _as_oracle_weights(w))
    y2, s2 = osb.block_forward_float(u, _as_oracle_weights(w2))
    assert np.abs(y2 - y1).max() <= 1e-5 * np.abs(y1).max()
    h1 = np.asarray(s1.h).reshape(nh, P, -1)
    h2 = np.asarray(s2.h).reshape(nh, P, -1)
    assert np.abs(reorder.permute_state(h1, plan) - h2).max() <= 1e-5 * np.abs(h1).max()
    inv = plan.inverse()
    assert np.array_equal(plan.pi[inv.pi], np.arange(d.d_inner))


def test_hadamard_transforms_are_orthogonal_fusions():
    """H_b H_b = b·I for the unnormalised butterflies, and the fused out_proj
    W·H̃ᵀ applied to H̃ y reproduces W y (H̃ = I_q ⊗ H_b / sqrt(b), the block-diagonal transform
    of LEDGER G9) — checked in float64 against the plain product, not against the oracle."""
    r = np.random.default_rng(6)
    for n, b in ((512, None), (5120, None), (384, 64)):
        v = torch.as_tensor(r.standard_normal((3, n)).astype(np.float32))
        bs = hadamard.block_size(n) if b is None else b
        twice = hadamard.fwht_blocked(hadamard.fwht_blocked(v, b), b)
        assert (twice - v * bs).abs().max() <= 1e-5 * (v * bs).abs().max()
    w = r.standard_normal((48, 384)).astype(np.float32)
    y = r.standard_normal((5, 384)).astype(np.float64)
    wf = hadamard.fuse_hadamard_out_proj(w, 384, 1).numpy().astype(np.float64)
    hy = hadamard.fwht_blocked(torch.as_tensor(y.astype(np.float32))).numpy().astype(np.float64) / np.sqrt(128)
    assert np.abs(hy @ wf.T - y @ w.T.astype(np.float64)).max() <= 1e-4 * np.abs(y @ w.T).max()


def test_weight_quantizers_round_trip_bounds():
    """Eq. 1: every code is in range, and dequantised weights
    are within half a step of the originals per scale group (per channel for W8, per 128-wide
    group for W4); the largest |w| of each group maps to ±(2^(b-1) - 1)."""
    r = np.random.default_rng(8)
    w = (r.standard_normal((64, 512)) * np.exp(r.uniform(-3, 1, (64, 1)))).astype(np.float32)
    for q, lo, hi in ((quantizer.quantize_weight_w8(w), -128, 127), (quantizer.quantize_weight_w4(w, 128), -8, 7)):
        c = _np(q.payload).astype(np.float64)
        s = _np(q.layout.expand(w.shape)).astype(np.float64)   # the scale of every element
        assert c.min() >= lo and c.max() <= hi
        assert np.all(np.abs(c * s - w) <= s / 2 * (1 + 1e-6))
        # the group's largest |w| lands on the top code (max|w| / (2^(b-1) - 1) is the scale)
        top = np.abs(c).reshape(64, -1, 128 if hi == 7 else 512).max(-1)
        assert np.all(top == hi)


# ---------------------------------------------------------------- GPTQ (acceptance 9)
def _proxy_loss(w, wq, X):
    d = X.astype(np.float64) @ (w.astype(np.float64) - wq.astype(np.float64)).T
    return float((d * d).sum())


def _deq(q):
    return _np(quantizer.dequantize(q)).astype(np.float64)


def test_gptq_spec_examples():
    """a 1x1 weight and a diagonal calibration covariance (orthogonal input
    columns, zero off-diagonal Hessian) give exactly the round-to-nearest codes and scales."""
    r = np.random.default_rng(0)
    w1 = np.array([[0.37]], np.float32)
    g1 = quantizer.gptq_quantize_weight(w1, r.standard_normal((3, 1)).astype(np.float32), 4, 1, device="cpu")
    rt = quantizer.quantize_weight_w4(w1, 1)
    assert torch.equal(g1.payload.cpu(), rt.payload) and np.array_equal(_deq(g1), _deq(rt))
    w = r.standard_normal((6, 16)).astype(np.float32)
    X = np.diag(r.uniform(0.5, 2.0, 16)).astype(np.float32)   # XᵀX diagonal
    for group in (16, 8):
        g = quantizer.gptq_quantize_weight(w, X, 4, group, device="cpu")
        rt = quantizer.quantize_weight_w4(w, group)
        assert torch.equal(g.payload.cpu(), rt.payload), group
        assert np.array_equal(_np(g.extra["s_group"]).reshape(-1), _np(rt.extra["s_group"]).reshape(-1))


@pytest.mark.parametrize("n,rows,group", [(8, 4, 8), (32, 8, 32), (64, 16, 16)])
def test_gptq_beats_rtn_on_the_proxy_loss(n, rows, group):
    """SPEC.md:154 / acceptance 9: the GPTQ proxy loss ||WX - ŴX||² is <= the RTN one in >= 18 of
    20 seeded trials (random n x n layer, `rows` calibration rows)."""
    wins = 0
    for seed in range(20):
        r = np.random.default_rng(100 + seed)
        w = r.standard_normal((n, n)).astype(np.float32)
        X = r.standard_normal((rows, n)).astype(np.float32)
        g = quantizer.gptq_quantize_weight(w, X, 4, group, device="cpu")
        rt = quantizer.quantize_weight_w4(w, group)
        wins += _proxy_loss(w, _deq(g), X) <= _proxy_loss(w, _deq(rt), X) * (1 + 1e-9)
        assert _np(g.payload).min() >= -8 and _np(g.payload).max() <= 7
    assert wins >= 18, wins


def test_gptq_singular_hessian_falls_back_to_rtn():
    """a Hessian still singular after damping (all-zero calibration, damp 0) is
    reported and the layer is rounded to nearest."""
    w = np.random.default_rng(1).standard_normal((4, 8)).astype(np.float32)
    with pytest.warns(RuntimeWarning):
        g = quantizer.gptq_quantize_weight(w, np.zeros((2, 8), np.float32), 4, 8, damp_ratio=0.0, device="cpu")
    assert torch.equal(g.payload.cpu(), quantizer.quantize_weight_w4(w, 8).payload)


@pytest.mark.parametrize("profile", ["W4A16", "W4A8"])
@pytest.mark.parametrize("dims", [TINY2, TINY1], ids=["mamba2", "mamba1"])
def test_pipeline_gptq_toggle_lowers_projection_loss(profile, dims):
    """The Table 7 "GPTQ" toggle: with gptq=True the 4-bit projections
    are rounded by GPTQ on calibration rows mapped into each weight's column basis (reordered,
    Hadamard-rotated out_proj input for A8, cluster-scaled x_proj input); on those rows the
    reconstruction loss ||X Wᵀ - X Ŵᵀ||² is no larger than round-to-nearest's, for every
    projection of the block."""
    d = Dims(*dims)
    fm = cli.cmd_gen_toy(d, 1, 3, 97)
    toks = cli.calib_tokens(97, 4, 24)
    stats = calibrate.collect_stats(fm, toks, device="cpu", keep_rows=96)
    qr = cli.quantize_block(fm.blocks[0], stats[0], profile)
    qg = cli.quantize_block(fm.blocks[0], stats[0], profile, gptq=True)
    rows = stats[0]["_rows"]
    pi = torch.as_tensor(qr.extra["plan"].pi)

    def deq(ql):
        return ql.codes.astype(np.float64) * np.repeat(ql.s_group.astype(np.float64), ql.group, axis=1)

    def loss(ql, X, w_ref):
        X = X.double().cpu().numpy()
        e = X @ (w_ref - deq(ql)).T
        return float((e * e).sum())

    X_out = rows["r"][:, pi]
    if profile == "W4A8":
        X_out = hadamard.fwht_blocked(X_out, d.had_block)
    pairs = [("in_proj", rows["u"]), ("out_proj", X_out)]
    if d.variant == "mamba1":
        pairs.append(("dt_proj", rows["dt_low"]))
    for name, X in pairs:
        w = _float_weight(fm.blocks[0], qr, name, d, profile)
        assert loss(getattr(qg, name), X, w) <= loss(getattr(qr, name), X, w) * (1 + 1e-9), name


def _float_weight(blk, qb, name, d, profile):
    """The float weight a QBlock projection was rounded from, in its column basis (reordered,
    Hadamard-fused out_proj for the A8 profiles)."""
    w = reorder.apply_reorder(blk, qb.extra["plan"])
    if name == "out_proj" and profile != "W4A16":
        b = d.had_block
        return (hadamard.fuse_hadamard_out_proj(w.out_proj, d.d_inner, 1, b).numpy() / np.float32(np.sqrt(b))).astype(
            np.float64)
    return np.asarray(getattr(w, name), np.float64)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_acceptance10_table7_ablation_monotone(seed):
    """SPEC.md acceptance 10 / :617: the five Table 7 toggle rows of the W4A8 pipeline, in the
    paper's order -- fail (no Hadamard) < PerG + Had < + GPTQ < + PerSG < + SnC -- give strictly
    improving block-output SQNR on the outlier toy model (gen-toy: heavy-tailed x channels, B / C
    state groups of different magnitude, outlier channels of the gated-norm output), and the
    no-Hadamard row is the minimum.  Quantized with the product pipeline, evaluated with the
    oracle's quantized block forward against the float block on held-out tokens."""
    from oracle import pipeline as opl
    from oracle import qblock as oq
    from oracle import ssm_block as osb
    dims = ("mamba2", 128, 256, 32, 16, 16, 4, 4)
    d = Dims(*dims)
    fm = cli.cmd_gen_toy(d, 1, seed, 64)
    stats = calibrate.collect_stats(fm, cli.calib_tokens(64, 8, 32), device="cpu", keep_rows=256)
    ofm = opl.cmd_gen_toy(osb.Dims(*dims), 1, seed, 64)
    ev = opl.calib_tokens(64, 2, 48, seed=9)
    u = osb.rmsnorm(ofm.embedding[ev[0]], ofm.layer_norms[0])
    ref, _ = osb.block_forward_float(u, ofm.blocks[0], fast=True)
    rows = [dict(hadamard=False, gptq=False, persg=False, snc=False),   # "fail"
            dict(hadamard=True, gptq=False, persg=False, snc=False),    # PerG + Had
            dict(hadamard=True, gptq=True, persg=False, snc=False),     # + GPTQ
            dict(hadamard=True, gptq=True, persg=True, snc=False),      # + PerSG
            dict(hadamard=True, gptq=True, persg=True, snc=True)]       # + SnC (the full pipeline)
    sq = []
    for kw in rows:
        p = cli.quantize_block(fm.blocks[0], stats[0], "W4A8", **kw)
        qb = oq.QBlock(osb.Dims(*dims), p.profile, oq.QLinear(**vars(p.in_proj)), oq.QLinear(**vars(p.out_proj)),
                       p.conv_weight, p.conv_bias, p.a_log, p.d_param, p.dt_bias, p.norm_weight, p.head_group,
                       s_u=p.s_u, in_out_scale=p.in_out_scale, conv_in_scale=p.conv_in_scale,
                       conv_out_scale=p.conv_out_scale, state_scale=p.state_scale, s_y=p.s_y, hadamard=p.hadamard)
        out, _ = oq.block_forward_quantized(u, qb)
        sq.append(10 * np.log10((ref ** 2).sum() / ((out - ref) ** 2).sum()))
    assert all(b > a for a, b in zip(sq, sq[1:])), sq
    assert sq[0] == min(sq)
