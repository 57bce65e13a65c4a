"""CPU: pin the oracle before trusting it.

1. Golden vectors produced by the SHIPPED reference (`tests/golden/make_golden.py`
   runs `pkg/src/ssmquant/tensor.py`): the oracle's `matmul` must match 0-ULP and its
   exact `int_gemm` must match on integer-valued operands.
2. Every numeric [TRIVIAL]/[DERIVED] example of SPEC.md on the hot path,
   each test citing its SPEC line.
3. SPEC acceptance criteria 1, 2, 3, 4, 5, 6, 7, 8, 12, 13, at
   sizes that finish in seconds.
"""
import json
import os

import numpy as np
import pytest

from oracle import calibrate as cal
from oracle import hadamard as had
from oracle import quantizer as qz
from oracle import reorder as ro
from oracle import ssm_block as sb
from oracle import tensor_core as tc
from oracle.errors import PipelineError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ reference goldens
def _gold():
    z = np.load(os.path.join(GOLD, "ref_matmul.npz"))
    names = sorted({k.rsplit(".", 1)[0] for k in z.files})
    return z, names


def test_golden_matmul_zero_ulp():
    z, names = _gold()
    assert len(names) >= 7
    for n in names:
        got = tc.matmul(z[f"{n}.a"], z[f"{n}.b"])
        assert got.dtype == np.float32
        assert np.array_equal(got.view(np.uint32), z[f"{n}.c"].view(np.uint32)), n


def test_golden_int_gemm_exact_on_integer_operands():
    z, names = _gold()
    for n in ("i8_8x512x12", "w4sg_4x256x6"):
        a, b, c = z[f"{n}.a"], z[f"{n}.b"], z[f"{n}.c"]
        acc = tc.int_gemm(a.astype(np.int64), b.astype(np.int64))
        # the reference returns f32 of the exact sum (D2): equal after the same rounding
        assert np.array_equal(acc.astype(np.float32), c)
        # and the exact sum itself equals a pure-integer triple loop
        assert np.array_equal(acc, a.astype(np.int64) @ b.astype(np.int64))


def test_golden_meta_reference_behaviour():
    with open(os.path.join(GOLD, "ref_meta.json")) as f:
        m = json.load(f)
    assert m["make_rng_raises"].startswith("ValueError")          # defect D1, fixed in oracle/product
    assert m["matmul_shape_error_is_valueerror"]
    for s, vals in m["fixed_rng_first_u64"].items():
        args = tuple(int(v) for v in s.strip("()").split(",") if v.strip())
        assert [int(v) for v in tc.make_rng(*args).integers(0, 2**63, 4)] == vals
    from oracle import errors as oe
    for n, bases in m["errors_hierarchy"].items():
        assert [b.__name__ for b in getattr(oe, n).__mro__[1:]] == bases


# ------------------------------------------------------------------ tensor_core
def test_matmul_spec_examples():
    assert np.array_equal(tc.matmul([[1, 2], [3, 4]], [[5], [6]]), [[17], [39]])
    assert np.array_equal(tc.matmul(np.zeros((1, 0)), np.zeros((0, 1))), [[0]])
    with pytest.raises(ValueError):
        tc.matmul(np.zeros((2, 3)), np.zeros((2, 3)))


def test_u4_packing_spec():
    assert tc.pack_u4([3, -2]).tolist() == [0xE3]
    v = np.arange(-8, 8).repeat(2).reshape(4, 8)
    assert np.array_equal(tc.unpack_u4(tc.pack_u4(v)), v)
    with pytest.raises(ValueError):
        tc.pack_u4([8, 0])


def test_archive_roundtrip_and_bytes(tmp_path):
    p = str(tmp_path / "a.bin")
    tc.archive_write({"w": np.zeros((2, 2), np.float32), "x": np.array([1.5], np.float32),
                      "q": ("u4packed", np.array([3, -2])), "i": np.array([-128, 127], np.int8),
                      "meta": {"k": [1, 2]}}, p)
    back = tc.archive_read(p)
    assert np.array_equal(back["w"], np.zeros((2, 2))) and back["meta"] == {"k": [1, 2]}
    assert back["q"].tolist() == [3, -2] and back["i"].tolist() == [-128, 127]
    raw = open(p, "rb").read()
    assert bytes([0x00, 0x00, 0xC0, 0x3F]) in raw
    assert bytes([0xE3]) in raw
    tc.archive_write({}, p)
    assert tc.archive_read(p) == {}
    tc.archive_write({"w": np.ones(4, np.float32)}, p)
    with open(p, "r+b") as f:
        f.truncate(len(open(p, "rb").read()) - 2)
    with pytest.raises(ValueError, match="blob shorter"):
        tc.archive_read(p)


# ------------------------------------------------------------------ quantizer
def test_compute_scale_and_quantize_spec():
    x = np.array([2.54, -1.27, 0.0], np.float32)
    s = qz.compute_scale(x, 8)
    assert np.isclose(s, 0.02)
    assert qz.compute_scale(np.zeros(5), 8) == 1.0
    assert qz.compute_scale([7.0], 4) == 1.0
    q = qz.quantize(x, qz.ScaleLayout("PerTensor", np.float32(0.02)), 8)
    assert q.payload.tolist() == [127, -64, 0]
    assert qz.quantize_codes([1000.0], np.float32(1.0 / 127), 8).tolist() == [127]
    s4 = np.float32(0.37)
    lat = (s4 * np.arange(-8, 8, dtype=np.float32)).astype(np.float32)
    assert qz.quantize_codes(lat, s4, 4).tolist() == list(range(-8, 8))
    dq = qz.dequantize(qz.QTensor((1,), 8, np.array([127], np.int8), qz.ScaleLayout("PerTensor", np.float32(0.02))))
    assert np.isclose(dq[0], 2.54)
    assert qz.fuse_scales(0.02, 1.0, 0.04) == np.float32(0.5)
    assert qz.fuse_scales(0.3, 1.0, 0.3) == 1.0


@pytest.mark.parametrize("bits", [4, 8])
def test_acceptance1_roundtrip_error(bits):
    """|dequant(quant(x)) - x| <= s/2 for 1e5 in-range values."""
    r = tc.make_rng(1, bits)
    s = np.float32(0.013)
    hi = (2 ** (bits - 1) - 1) * s
    x = r.uniform(-hi, hi, 100_000).astype(np.float32)
    q = qz.quantize(x, qz.ScaleLayout("PerTensor", s), bits)
    err = np.abs(qz.dequantize(q) - x)
    assert (err <= s / 2 * (1 + 1e-6)).all()


def test_quantize_scale_homogeneous_codes():
    """quantize(αx) with scale αs → identical integer payload (α a power of 2 keeps f32 exact)."""
    r = tc.make_rng(2)
    x = r.standard_normal(1000).astype(np.float32)
    s = qz.compute_scale(x, 8)
    for a in (0.25, 2.0, 64.0):
        assert np.array_equal(qz.quantize_codes(x * np.float32(a), s * np.float32(a), 8), qz.quantize_codes(x, s, 8))


def test_fused_scale_gemm_vs_float():
    """8-bit GEMM with fused scales vs float GEMM on 16x16, rel err <= 2%."""
    r = tc.make_rng(3)
    X = r.standard_normal((16, 16)).astype(np.float32)
    W = r.standard_normal((16, 16)).astype(np.float32)
    sx, sw = qz.compute_scale(X, 8), qz.compute_scale(W, 8)
    acc = tc.int_gemm(qz.quantize_codes(X, sx, 8), qz.quantize_codes(W, sw, 8))
    ref = tc.matmul(X, W)
    got = acc.astype(np.float32) * (sx * sw)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 0.02


def test_weight_quantizers_layouts():
    r = tc.make_rng(4)
    w = (r.standard_normal((6, 256)) * np.exp(r.uniform(-2, 2, (1, 256)))).astype(np.float32)
    q8 = qz.quantize_weight_w8(w)
    assert np.abs(qz.dequantize(q8) - w).max() <= q8.extra["s_ch"].max() / 2 * 1.0001
    q4 = qz.quantize_weight_w4_group(w, 128)
    assert q4.payload.min() >= -8 and q4.payload.max() <= 7
    err = np.abs(qz.dequantize(q4) - w)
    assert (err <= np.repeat(q4.extra["s_group"], 128, axis=1) / 2 * 1.0001).all()
    qa = qz.quantize_weight_w4a8(w, 128)     # LEDGER G11: W4A8 weights are the SPEC PerGroup format
    assert np.array_equal(qa.payload, q4.payload) and np.array_equal(qa.extra["s_group"], q4.extra["s_group"])


def test_w4a8_zero_group_keeps_row_precision():
    """an all-zero 128-group must not coarsen the rest of its row (it did under the
    round-1 progressive scales); per-group SPEC scales keep every group at its own absmax/7."""
    r = tc.make_rng(41)
    w = (r.standard_normal((4, 512)) * 0.02).astype(np.float32)
    w[1, 128:256] = 0.0
    qa = qz.quantize_weight_w4a8(w, 128)
    assert qa.extra["s_group"][1, 1] == np.float32(1.0)                      # SPEC.md:117 zero slice
    err = np.abs(qz.dequantize(qa) - w)
    assert (err <= np.repeat(qa.extra["s_group"], 128, axis=1) / 2 * 1.0001).all()
    assert np.abs(qa.payload[1, :128]).max() == 7                             # the row keeps full range


def test_w4a8_promotion_order_and_splits():
    """qlinear_a8 (W4A8) == the documented promotion: per split, ascending groups from 0, then
    the split partials in order; splits=1 vs 2 differ only by f32 re-association."""
    from oracle import qblock as oq
    r = tc.make_rng(42)
    M, N, K = 5, 7, 512
    a = r.integers(-128, 128, (M, K)).astype(np.int8)
    codes = r.integers(-8, 8, (N, K)).astype(np.int8)
    s = r.uniform(1e-3, 1e-2, (N, K // 128)).astype(np.float32)
    ql = oq.QLinear("w4a8", codes, s_group=s, group=128)
    y1, acc = oq.qlinear_a8(a, ql, np.float32(0.5), splits=1)
    assert np.array_equal(acc, tc.int_gemm(a, codes.T))
    from fractions import Fraction

    def round_f32(x: Fraction) -> np.float32:   # correctly rounded (ties to even), no double rounding
        c = np.float32(float(x))
        cands = [np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))]
        err = [abs(Fraction(float(v)) - x) for v in cands]
        best = min(err)
        tied = [v for v, e in zip(cands, err) if e == best]
        return min(tied, key=lambda v: int(np.asarray(v).view(np.int32)) & 1)

    for m in range(M):                       # exact rational fma, rounded to f32 once per group
        for n in range(N):
            p = np.float32(0)
            for g in range(4):
                acc = int(tc.int_gemm(a[m:m + 1, g * 128:(g + 1) * 128], codes[n:n + 1, g * 128:(g + 1) * 128].T)[0, 0])
                p = round_f32(Fraction(float(s[n, g])) * acc + Fraction(float(p)))
            assert y1[m, n] == np.float32(p * np.float32(0.5))
    y2, _ = oq.qlinear_a8(a, ql, np.float32(0.5), splits=2)
    assert np.allclose(y1, y2, rtol=1e-6, atol=1e-6 * np.abs(y1).max())


# ------------------------------------------------------------------ hadamard
def test_fwht_spec_examples():
    assert had.fwht(np.array([3.5], np.float32), had.HadamardPlan(1)).tolist() == [3.5]
    assert had.fwht(np.array([1, 0, 0, 0], np.float32), had.HadamardPlan(4)).tolist() == [1, 1, 1, 1]  # :201
    r = tc.make_rng(5)
    v = r.standard_normal((3, 64)).astype(np.float32)
    p = had.HadamardPlan(64, "sqrt")
    assert np.allclose(had.fwht(had.fwht(v, p), p), v, rtol=1e-6, atol=1e-6)


def test_acceptance2_fwht_vs_dense():
    """SPEC.md:637 (and :232-233)."""
    r = tc.make_rng(6)
    n = 2
    while n <= 1024:
        H = had.hadamard_matrix(n)
        assert np.array_equal(H @ H.T, n * np.eye(n, dtype=np.int64))
        v = r.standard_normal((4, n)).astype(np.float32)
        dense = v.astype(np.float64) @ H.T
        got = had.fwht(v, had.HadamardPlan(n))
        assert np.abs(got - dense).max() <= 1e-6 * np.abs(dense).max() * np.sqrt(n) + 1e-6
        n *= 2


def test_hadamard_fusion_examples():
    assert np.allclose(had.fuse_hadamard_out_proj(np.eye(8, dtype=np.float32), 8, 8), np.eye(8), atol=1e-6)  # :209
    assert np.allclose(had.fuse_hadamard_in_proj(np.ones((1, 2), np.float32)), [[np.sqrt(2), 0]], atol=1e-6)  # :219
    assert not had.fuse_hadamard_out_proj(np.zeros((4, 4), np.float32), 4, 4).any()      # :211
    r = tc.make_rng(7)
    W = r.standard_normal((4, 4)).astype(np.float32)
    x = r.standard_normal(4).astype(np.float32)
    H = had.hadamard_matrix(4) / 2.0
    Wf = had.fuse_hadamard_out_proj(W, 4, 4)
    assert np.allclose(H.T @ (Wf @ (H @ x)), W @ x, atol=1e-5)                            # :210


def test_hadamard_quantize_spec():
    r = tc.make_rng(8)
    y = r.standard_normal((5, 128)).astype(np.float32)
    t = had.fwht(y, had.HadamardPlan(128))
    s = qz.compute_scale(t, 8)
    one = had.hadamard_quantize(y, had.HadamardPlan(128, "none", s), 8)
    two = qz.quantize(t, qz.ScaleLayout("PerTensor", s), 8).payload
    assert np.array_equal(one, two)
    assert not had.hadamard_quantize(np.zeros((2, 64), np.float32), had.HadamardPlan(64, "none", 0.1), 8).any()
    out = np.zeros(64, np.float32)
    out[0] = 100.0
    hv = had.fwht(out, had.HadamardPlan(64, "sqrt"))
    assert np.isclose(np.abs(out).max() / np.abs(hv).max(), 8.0)


def test_blocked_hadamard_non_pow2_orthogonal():
    """LEDGER G9: I_q ⊗ H_b for n = 5120 style widths (here 40 = 5·8)."""
    M = had.blocked_matrix(40)
    assert np.array_equal(M @ M.T, 8 * np.eye(40, dtype=np.int64))
    r = tc.make_rng(9)
    v = r.standard_normal((2, 40)).astype(np.float32)
    assert np.allclose(had.fwht_blocked(v), v @ M.T, atol=1e-5)


# ------------------------------------------------------------------ ssm_block
def _toy_dims(variant="mamba2"):
    if variant == "mamba2":
        return sb.Dims("mamba2", 64, 128, 16, 8, 16, 2, 4)          # SPEC.md:348 toy defaults
    return sb.Dims("mamba1", 64, 128, 16, 1, 128, 1, 4, dt_rank=8)


def _toy_block(seed=0, variant="mamba2"):
    from oracle.pipeline import gen_block
    return gen_block(_toy_dims(variant), seed, 0)


def test_conv_spec_examples():
    r = tc.make_rng(10)
    x = r.standard_normal((7, 5)).astype(np.float32)
    y, _ = sb.causal_conv1d(x, np.ones((5, 1), np.float32), np.zeros(5, np.float32))
    assert np.array_equal(y, sb.silu(x))
    w = r.standard_normal((5, 4)).astype(np.float32)
    b = r.standard_normal(5).astype(np.float32)
    full, _ = sb.causal_conv1d(x, w, b)
    cache, steps = None, []
    for t in range(7):
        o, cache = sb.causal_conv1d(x[t:t + 1], w, b, cache)
        steps.append(o)
    assert np.allclose(np.concatenate(steps), full, rtol=1e-6, atol=1e-7)
    z, _ = sb.causal_conv1d(np.zeros((3, 5), np.float32), w, b)
    assert np.allclose(z, np.broadcast_to(sb.silu(b), (3, 5)))


def test_discretize_and_scalar_scan_spec():
    dA, dt = sb.discretize(np.zeros((1, 1), np.float32), np.zeros(1, np.float32), np.array([-1.0], np.float32))
    assert np.isclose(dt[0, 0], np.log(2)) and np.isclose(dA[0, 0], 0.5)
    dA2, dt2 = sb.discretize(np.array([[-1e4]], np.float32), np.zeros(1, np.float32), np.array([-1.0], np.float32))
    assert dt2[0, 0] < 1e-30 and dA2[0, 0] == 1.0
    x = np.ones((1, 1, 1), np.float32)
    B = C = np.ones((1, 1, 1), np.float32)
    y, h = sb.selective_scan(x, dA, dt, B, C, np.zeros(1, np.float32))
    assert np.isclose(h[0, 0, 0], np.log(2)) and np.isclose(y[0, 0, 0], np.log(2))


def _rand_scan_inputs(r, T, nh=4, P=8, G=2, N=8):
    x = r.standard_normal((T, nh, P)).astype(np.float32)
    dt = sb.softplus(r.standard_normal((T, nh)).astype(np.float32) - 1)
    A = -np.exp(r.uniform(0, 1.5, nh)).astype(np.float32)
    dA = np.exp(dt * A).astype(np.float32)
    B = r.standard_normal((T, G, N)).astype(np.float32)
    C = r.standard_normal((T, G, N)).astype(np.float32)
    D = r.standard_normal(nh).astype(np.float32)
    z = r.standard_normal((T, nh, P)).astype(np.float32)
    return x, dA, dt, B, C, D, z


def test_acceptance5_ssd_equals_scan():
    """SPEC.md:640 (T subsampled from 1..128 for runtime), chunk ∈ {1,3,16,T}."""
    r = tc.make_rng(11)
    for T in (1, 2, 5, 16, 17, 63, 128):
        args = _rand_scan_inputs(r, T)
        ys, hs = sb.selective_scan(*args)
        for ch in sorted({1, 3, 16, T}):
            yc, hc = sb.ssd_chunked(*args, chunk=ch)
            sc = np.abs(ys).max()
            assert np.abs(yc - ys).max() <= 1e-4 * sc, (T, ch)
            assert np.abs(hc - hs).max() <= 1e-4 * np.abs(hs).max()


def test_scan_memoryless_and_single_step():
    r = tc.make_rng(12)
    x, dA, dt, B, C, D, _ = _rand_scan_inputs(r, 3)
    y, _ = sb.selective_scan(x, np.zeros_like(dA), dt, B, C, D)
    hg = np.arange(4) // 2
    for t in range(3):
        ref = np.einsum("hn,hn->h", C[t][hg], B[t][hg])[:, None] * dt[t][:, None] * x[t] + D[:, None] * x[t]
        assert np.allclose(y[t], ref, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("variant", ["mamba2", "mamba1"])
def test_acceptance5_decode_equals_prefill(variant):
    """stateful single-token stepping over 32 steps == full forward (≤1e-5)."""
    w = _toy_block(1, variant)
    r = tc.make_rng(13)
    u = r.standard_normal((32, 64)).astype(np.float32)
    full, _ = sb.block_forward_float(u, w, fast=True)
    st, outs = None, []
    for t in range(32):
        o, st = sb.block_forward_float(u[t:t + 1], w, st, fast=True)
        outs.append(o)
    step = np.concatenate(outs)
    assert np.abs(step - full).max() <= 1e-5 * np.abs(full).max()


def test_block_zero_input_zero_output():
    w = _toy_block(2)
    w = w.copy(conv_bias=np.zeros_like(w.conv_bias))
    out, _ = sb.block_forward_float(np.zeros((4, 64), np.float32), w, fast=True)
    assert not out.any()


def test_acceptance6_channel_order_preservation():
    """permuting x-channels (with matching rows) leaves output unchanged."""
    w = _toy_block(3)
    d = w.dims
    r = tc.make_rng(14)
    u = r.standard_normal((12, 64)).astype(np.float32)
    ref, _ = sb.block_forward_float(u, w, fast=True)
    for k in range(20):
        pr = tc.make_rng(15, k)
        head_perm = pr.permutation(d.n_heads)
        cperm = np.stack([pr.permutation(d.head_dim) for _ in range(d.n_heads)])
        cmap = cal.ClusterMap(head_perm, cperm, np.array([0, d.n_heads]), np.array([[0, d.head_dim]]),
                              np.ones((1, 1), np.float32))
        w2 = ro.apply_reorder(w, ro.build_reorder_plan(cmap, d))
        out, _ = sb.block_forward_float(u, w2, fast=True)
        assert np.abs(out - ref).max() <= 1e-5 * np.abs(ref).max()


# ------------------------------------------------------------------ calibrate
def test_sort_and_cluster_spec_example():
    """4 heads {[10,1],[0.1,0.05],[9,1.2],[0.12,0.04]}, m=2 → {0,2},{1,3}."""
    st = cal.CalibStats(np.array([[10, 1], [0.1, 0.05], [9, 1.2], [0.12, 0.04]], np.float32).reshape(-1), 1)
    cm = cal.sort_and_cluster(st, 4, 2, m=2, n=1)
    groups = [sorted(cm.head_perm[cm.head_group_bounds[i]:cm.head_group_bounds[i + 1]].tolist()) for i in range(2)]
    assert sorted(groups) == [[0, 2], [1, 3]]
    cm1 = cal.sort_and_cluster(st, 4, 2, m=1, n=1)
    assert cm1.scales.shape == (1, 1) and np.isclose(cm1.scales[0, 0], 10 / 127)


def test_cluster_map_invariants():
    r = tc.make_rng(16)
    mx = (np.exp(r.uniform(-3, 3, (8, 16))) * np.exp(r.uniform(-2, 2, (8, 1)))).astype(np.float32)
    cm = cal.sort_and_cluster(cal.CalibStats(mx.reshape(-1), 1), 8, 16, 4, 4)
    assert sorted(cm.head_perm.tolist()) == list(range(8))
    for h in range(8):
        assert sorted(cm.channel_perm[h].tolist()) == list(range(16))
        assert (np.diff(mx[h][cm.channel_perm[h]]) <= 0).all()
    assert (np.diff(cm.head_group_bounds) > 0).all() and cm.head_group_bounds[-1] == 8
    assert (np.diff(cm.channel_group_bounds, axis=1) > 0).all()
    # per-group max reproduction within one step
    cells = cm.cell_of_new()
    pl = ro.build_reorder_plan(cm, sb.Dims("mamba2", 8, 128, 8, 8, 16, 1))
    mx_new = mx.reshape(-1)[pl.pi]
    for c in range(cm.m * cm.n):
        gmax = mx_new[cells == c].max()
        s = cm.scales.reshape(-1)[c]
        assert abs(127 * s - gmax) <= s
    assert cal.sort_and_cluster(cal.CalibStats(mx.reshape(-1), 1), 8, 16, 4, 4).head_perm.tolist() == \
        cm.head_perm.tolist()                                                              # SPEC.md:424 determinism


def test_state_group_scales_spec():
    sB = cal.CalibStats(np.array([10.0] * 4 + [0.1] * 4, np.float32), 1)
    g = cal.build_state_group_scales(sB, sB, 2, 4)
    assert np.allclose(g.scales_B, [10 / 127, 0.1 / 127])
    g1 = cal.build_state_group_scales(sB, sB, 1, 8)
    assert np.allclose(g1.scales_B, [10 / 127])
    u = cal.CalibStats(np.full(8, 3.0, np.float32), 1)
    assert np.all(cal.build_state_group_scales(u, u, 4, 2).scales_C == np.float32(3 / 127))


def test_calibrate_site_scale_spec():
    assert np.isclose(cal.calibrate_site_scale(cal.CalibStats(np.array([2.54], np.float32), 1)), 0.02)  # :417
    assert cal.calibrate_site_scale(cal.CalibStats(np.zeros(3, np.float32), 1)) == 1.0              # :419
    v = np.ones(10_000, np.float32)
    v[17] = 1e6
    st = cal.stats_of(v[:, None], (1,), keep_values=True)
    s = cal.calibrate_site_scale(st, 8, clip_percentile=99.9)
    assert np.isclose(s, 1 / 127)                                                          # :418
    a = cal.stats_of(np.abs(np.arange(6, dtype=np.float32)).reshape(3, 2), (2,))
    b = cal.stats_of(np.full((2, 2), 7, np.float32), (2,))
    assert np.array_equal(a.merge(b).channel_max, b.merge(a).channel_max)                  # :391


def test_acceptance7_sort_and_cluster_benefit():
    """clustered m=n=4 MSE ≤ 0.5× per-tensor MSE (averaged over seeds)."""
    ratios = []
    for seed in range(5):
        r = tc.make_rng(17, seed)
        nh, P = 8, 16
        ch = np.exp(r.uniform(np.log(0.01), np.log(10), (nh, P))).astype(np.float32)
        x = (r.standard_t(3, (64, nh, P)) * ch).astype(np.float32).reshape(64, -1)
        st = cal.stats_of(x, (nh * P,))
        cm = cal.sort_and_cluster(st, nh, P, 4, 4, seed)
        pl = ro.build_reorder_plan(cm, sb.Dims("mamba2", 8, nh * P, 8, nh, P, 1))
        xr = x[:, pl.pi]
        s_cells = cm.scales.reshape(-1)[cm.cell_of_new()]
        e_cl = ((qz.quantize_codes(xr, s_cells[None], 8) * s_cells - xr) ** 2).mean()
        s_t = qz.compute_scale(x, 8)
        e_t = ((qz.quantize_codes(x, s_t, 8) * s_t - x) ** 2).mean()
        ratios.append(e_cl / e_t)
    assert np.mean(ratios) <= 0.5


def test_acceptance8_per_state_group_benefit():
    r = tc.make_rng(18)
    B = r.standard_normal((256, 2, 8)).astype(np.float32)
    B[:, 1] *= 0.05
    st = cal.stats_of(B.reshape(256, -1), (16,))
    g = cal.build_state_group_scales(st, st, 2, 8)
    s_g = np.repeat(g.scales_B, 8)
    e_g = ((qz.quantize_codes(B.reshape(256, -1), s_g[None], 8) * s_g - B.reshape(256, -1)) ** 2).mean()
    s_t = qz.compute_scale(B, 8)
    e_t = ((qz.quantize_codes(B, s_t, 8) * s_t - B) ** 2).mean()
    assert e_g < e_t


# ------------------------------------------------------------------ reorder
def test_reorder_plan_spec_example():
    cm = cal.ClusterMap(np.array([1, 0]), np.array([[1, 0], [1, 0]]), np.array([0, 2]), np.array([[0, 2]]),
                        np.ones((1, 1), np.float32))
    assert ro.build_reorder_plan(cm, sb.Dims("mamba2", 4, 4, 4, 2, 2, 1)).pi.tolist() == [3, 2, 1, 0]  # :464
    ident = cal.ClusterMap(np.arange(2), np.tile(np.arange(2), (2, 1)), np.array([0, 2]), np.array([[0, 2]]),
                           np.ones((1, 1), np.float32))
    assert ro.build_reorder_plan(ident, sb.Dims("mamba2", 4, 4, 4, 2, 2, 1)).pi.tolist() == [0, 1, 2, 3]  # :463


@pytest.mark.parametrize("variant", ["mamba2", "mamba1"])
def test_acceptance4_reorder_invariance_and_inverse(variant):
    """SPEC.md:639 (10 random ClusterMaps per variant for runtime)."""
    w = _toy_block(4, variant)
    d = w.dims
    nh, P = (d.n_heads, d.head_dim) if variant == "mamba2" else (1, d.d_inner)
    r = tc.make_rng(19)
    u = r.standard_normal((10, 64)).astype(np.float32)
    ref, _ = sb.block_forward_float(u, w, fast=True)
    for k in range(10):
        pr = tc.make_rng(20, k)
        cm = cal.ClusterMap(pr.permutation(nh), np.stack([pr.permutation(P) for _ in range(nh)]),
                            np.array([0, nh]), np.array([[0, P]]), np.ones((1, 1), np.float32))
        plan = ro.build_reorder_plan(cm, d)
        w2 = ro.apply_reorder(w, plan)
        out, _ = sb.block_forward_float(u, w2, fast=True)
        assert np.abs(out - ref).max() <= 1e-5 * np.abs(ref).max()
        back = ro.apply_reorder(w2.copy(applied=()), plan.inverse())
        for f in ("in_proj", "conv_weight", "conv_bias", "a_log", "d_param", "dt_bias", "norm_weight", "out_proj"):
            assert np.array_equal(getattr(back, f), getattr(w, f)), f
        with pytest.raises(PipelineError):
            ro.apply_reorder(w2, plan)


def test_acceptance3_hadamard_block_invariance():
    """fused out_proj + online transform == unfused float block (≤1e-5), 10 toy blocks."""
    for seed in range(10):
        w = _toy_block(30 + seed)
        r = tc.make_rng(21, seed)
        u = r.standard_normal((6, 64)).astype(np.float32)
        ref, _ = sb.block_forward_float(u, w, fast=True)
        di = w.dims.d_inner
        wf = had.fuse_hadamard_out_proj(w.out_proj, di, 1)
        # block with fused weight and online normalised H on the out_proj input
        taps = {}
        sb.block_forward_float(u, w, fast=True, taps=taps)
        yh = had.fwht_blocked(taps["r"]) / np.float32(np.sqrt(had.block_size(di)))
        out = tc.matmul_fast(yh, wf.T)
        assert np.abs(out - ref).max() <= 1e-5 * np.abs(ref).max()


# ------------------------------------------------------------------ pipeline
def test_acceptance13_determinism_and_12_sizes(tmp_path):
    from oracle import pipeline as opl
    d = sb.Dims("mamba2", 64, 128, 16, 8, 16, 2, 4)
    a = opl.cmd_gen_toy(d, 2, seed=5, vocab=64)
    b = opl.cmd_gen_toy(d, 2, seed=5, vocab=64)
    for x, y in zip(a.blocks, b.blocks):
        assert np.array_equal(x.in_proj, y.in_proj) and np.array_equal(x.a_log, y.a_log)
        assert (x.A < 0).all()
    toks = opl.calib_tokens(64, 2, 16)
    q1 = opl.cmd_quantize(a, toks, "W4A8")
    q2 = opl.cmd_quantize(b, toks, "W4A8")
    for x, y in zip(q1.blocks, q2.blocks):
        assert np.array_equal(x.in_proj.codes, y.in_proj.codes)
        assert np.array_equal(x.extra["cmap"].head_perm, y.extra["cmap"].head_perm)
        assert np.array_equal(x.state_scale, y.state_scale)
    # size accounting direction: int4 payload is 1/8 of f32 bytes
    fl = sum(blk.in_proj.nbytes + blk.out_proj.nbytes for blk in a.blocks)
    q4 = sum(blk.in_proj.codes.size // 2 + 4 * blk.in_proj.s_group.size +
             blk.out_proj.codes.size // 2 + 4 * blk.out_proj.s_group.size for blk in q1.blocks)
    assert q4 <= 0.3 * fl


def test_quantized_block_sqnr_ordering():
    """SQNR(W8A8) > SQNR(W4A8) on the same toy model and inputs."""
    from oracle import pipeline as opl
    from oracle import qblock as oq
    d = sb.Dims("mamba2", 64, 128, 16, 8, 16, 2, 4)
    fm = opl.cmd_gen_toy(d, 1, seed=6, vocab=64)
    toks = opl.calib_tokens(64, 2, 24)
    u = sb.rmsnorm(fm.embedding[toks[0]], fm.layer_norms[0])
    ref, _ = sb.block_forward_float(u, fm.blocks[0], fast=True)
    stats = opl.collect_stats(fm, toks)
    sq = {}
    for prof in ("W8A8", "W4A8"):
        qb = opl.quantize_block(fm.blocks[0], stats[0], prof)
        out, _ = oq.block_forward_quantized(u, qb)
        sq[prof] = 10 * np.log10((ref ** 2).sum() / ((out - ref) ** 2).sum())
    assert sq["W8A8"] > sq["W4A8"] > 10
