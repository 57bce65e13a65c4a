"""Oracle: SPEC `[MODULE] cli_pipeline` gen-toy / quantize + the model wrapper (LEDGER G8).

TEST INFRASTRUCTURE ONLY.

Model (G8): pre-norm residual Mamba stack
    h = E[tok];  for l: h += block_l(rmsnorm(h, ln_l));  logits = head(rmsnorm(h, ln_f))
Head-to-toe: embedding per-row 8-bit, head per-group 4-bit
(W4A8, activation per-tensor 8-bit) in A8 plans; the block profile decides
each block's weights.

gen-toy: weights N(0,1/√fan_in); x-slice rows of in_proj get
per-channel log-uniform multipliers spanning 100× (channel persistence, Fig. 3);
a_log = log U[1,16] (A<0); dt_bias = softplus⁻¹(U[1e-3, 1e-1]); D = 1;
embedding rows Student-t(ν=3) with per-channel log-uniform scales.
Every tensor draws from make_rng(seed, layer, tensor_id).

quantize, fixed stage order: collect_stats (float model) →
sort_and_cluster → build_state_group_scales → reorder → Hadamard fusion of
out_proj (A8) → weight quantisation → activation-scale embedding.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from oracle import calibrate as cal
from oracle import hadamard as had
from oracle import reorder as ro
from oracle.qblock import QBlock, QState, block_forward_quantized, make_qlinear, qlinear_a8, zero_qstate
from oracle.quantizer import compute_scale, quantize_codes
from oracle.ssm_block import Dims, SsmBlockWeights, block_forward_float, rmsnorm, zero_state
from oracle.tensor_core import make_rng, matmul_fast

T_IN, T_CONV_W, T_CONV_B, T_ALOG, T_DTB, T_NORM, T_OUT, T_XPROJ, T_DTPROJ, T_MULT, T_BCG, T_NOUT = range(12)


def _gemm_group(k: int) -> int:
    return 128 if k % 128 == 0 else (32 if k % 32 == 0 else k)


def gen_block(d: Dims, seed: int, layer: int, n_layers: int = 1) -> SsmBlockWeights:
    r = lambda t: make_rng(seed, layer + 1, t)
    di, dm = d.d_inner, d.d_model
    inp = (r(T_IN).standard_normal((d.in_proj_out, dm)) / np.sqrt(dm)).astype(np.float32)
    mult = np.exp(r(T_MULT).uniform(np.log(0.1), np.log(10.0), di)).astype(np.float32)
    inp[di:2 * di] *= mult[:, None]
    if d.variant == "mamba2" and d.n_state_groups > 1:
        # state groups of different magnitude (B rows of group g scaled by a factor of 0.01-10x, C rows by its inverse):
        # what per-state-group B/C scales exploit (Fig. 3e-f; SPEC.md acceptance 8, 10)
        gn = d.n_state_groups * d.d_state
        gmul = np.exp(r(T_BCG).uniform(np.log(0.01), np.log(10.0), d.n_state_groups)).astype(np.float32)
        gm = np.repeat(gmul, d.d_state)
        inp[2 * di:2 * di + gn] *= gm[:, None]
        inp[2 * di + gn:2 * di + 2 * gn] /= gm[:, None]   # C inversely: every group's C·h stays O(1)
    K = d.conv_kernel
    conv_w = (r(T_CONV_W).standard_normal((d.conv_dim, K)) * 0.5 / np.sqrt(K)).astype(np.float32)
    conv_b = (r(T_CONV_B).standard_normal(d.conv_dim) * 0.05).astype(np.float32)
    dtv = r(T_DTB).uniform(1e-3, 1e-1, d.n_heads if d.variant == "mamba2" else di)
    dt_bias = (dtv + np.log(-np.expm1(-dtv))).astype(np.float32)
    if d.variant == "mamba2":
        a_log = np.log(r(T_ALOG).uniform(1, 16, d.n_heads)).astype(np.float32)
        dpar = np.ones(d.n_heads, np.float32)
    else:
        a_log = np.log(np.tile(np.arange(1, d.d_state + 1, dtype=np.float32), (di, 1))
                       * r(T_ALOG).uniform(0.5, 1.5, (di, 1))).astype(np.float32)
        dpar = np.ones(di, np.float32)
    norm = (1.0 + 0.1 * r(T_NORM).standard_normal(di)).astype(np.float32)
    # a few outlier channels of the gated-norm output (the out_proj input): what the Hadamard
    # rotation before the out_proj quantizer spreads out (§3.3; SPEC.md acceptance 10)
    hot = r(T_NOUT).choice(di, max(1, di // 64), replace=False)
    norm[hot] *= np.float32(100.0)
    out = (r(T_OUT).standard_normal((dm, di)) / np.sqrt(di) / np.sqrt(2 * n_layers)).astype(np.float32)
    xp = dtp = None
    if d.variant == "mamba1":
        R, N = d.dt_rank, d.d_state
        xp = (r(T_XPROJ).standard_normal((R + 2 * N, di)) / np.sqrt(di)).astype(np.float32)
        dtp = (r(T_DTPROJ).standard_normal((di, R)) / np.sqrt(R)).astype(np.float32)
    return SsmBlockWeights(d, inp, conv_w, conv_b, a_log, dpar, dt_bias, norm, out, xp, dtp)


@dataclass
class FloatModel:
    dims: Dims
    embedding: np.ndarray
    layer_norms: list
    blocks: list
    final_norm: np.ndarray
    head: np.ndarray


def cmd_gen_toy(d: Dims, n_blocks: int, seed: int = 0, vocab: int = 512) -> FloatModel:
    """SPEC.md:579-587 (returns the model; archive writing is the CLI's job)."""
    r = lambda t: make_rng(seed, 0, t)
    chs = np.exp(r(1).uniform(np.log(0.1), np.log(10.0), d.d_model))
    emb = (r(2).standard_t(3, (vocab, d.d_model)) * chs).astype(np.float32)
    lns = [(1.0 + 0.1 * make_rng(seed, 1000 + l, 0).standard_normal(d.d_model)).astype(np.float32)
           for l in range(n_blocks)]
    blocks = [gen_block(d, seed, l, n_blocks) for l in range(n_blocks)]
    fn = np.ones(d.d_model, np.float32)
    head = (r(3).standard_normal((vocab, d.d_model)) / np.sqrt(d.d_model)).astype(np.float32)
    return FloatModel(d, emb, lns, blocks, fn, head)


def calib_tokens(vocab: int, n_samples: int, seq_len: int, seed: int = 0) -> np.ndarray:
    return make_rng(seed, 7, 7).integers(0, vocab, (n_samples, seq_len))


def float_forward(model: FloatModel, tokens, taps=None, fast=True):
    """tokens [T] → logits [T×V]; taps[l] receives block l's calibration sites."""
    h = model.embedding[np.asarray(tokens)].astype(np.float32)
    for l, blk in enumerate(model.blocks):
        u = rmsnorm(h, model.layer_norms[l])
        t = {} if taps is not None else None
        out, _ = block_forward_float(u, blk, fast=fast, taps=t)
        if taps is not None:
            taps.append(t)
        h = (h + out).astype(np.float32)
    hf = rmsnorm(h, model.final_norm)
    if taps is not None:
        taps.append({"head_in": hf})
    return matmul_fast(hf, model.head.T)


def collect_stats(model: FloatModel, tokens, sites=None):
    """per layer, per site channel maxima over all samples."""
    L = len(model.blocks)
    d = model.dims
    stats = [dict() for _ in range(L + 1)]
    for s in range(tokens.shape[0]):
        taps = []
        float_forward(model, tokens[s], taps)
        for l in range(L + 1):
            for k, v in taps[l].items():
                v = np.asarray(v)
                ch = v.shape[1:] if k not in ("h",) else v.shape
                st = cal.stats_of(v[None] if k == "h" else v, ch)
                stats[l][k] = st if k not in stats[l] else stats[l][k].merge(st)
    return stats


@dataclass
class QuantModel:
    dims: Dims
    profiles: list
    emb_codes: np.ndarray
    emb_scale: np.ndarray
    layer_norms: list
    blocks: list
    final_norm: np.ndarray
    head: object
    s_head: np.float32
    extra: dict = field(default_factory=dict)


def quantize_block(blk: SsmBlockWeights, st: dict, profile: str, m=4, n=4, hadamard=True, reorder=True, seed=0):
    d = blk.dims
    di = d.d_inner
    if d.variant == "mamba2":
        nh, P = d.n_heads, d.head_dim
    else:
        nh, P = 1, d.d_inner
    cmap = cal.sort_and_cluster(st["x"], nh, P, m, n, seed)
    plan = ro.build_reorder_plan(cmap, d)
    w = ro.apply_reorder(blk, plan) if reorder else blk
    cells = cmap.cell_of_new()
    if not reorder:                      # clustered scales looked up in the original layout
        c0 = np.empty_like(cells)
        c0[plan.pi] = cells
        cells = c0
    a8 = profile in ("W8A8", "W4A8")
    kind = {"W8A8": "w8", "W4A8": "w4a8", "W4A16": "w4a16"}[profile]
    extra = {"cmap": cmap, "plan": plan}
    if not a8:
        qb = QBlock(d, profile, make_qlinear(w.in_proj, kind, _gemm_group(d.d_model)),
                    make_qlinear(w.out_proj, kind, _gemm_group(di)),
                    w.conv_weight, w.conv_bias, w.a_log, w.d_param, w.dt_bias, w.norm_weight, w.head_group,
                    extra=extra)
        if d.variant == "mamba1":
            qb.x_proj = make_qlinear(w.x_proj, kind, _gemm_group(di))
            qb.dt_proj = make_qlinear(w.dt_proj, kind, _gemm_group(d.dt_rank))
        return qb
    s_u = cal.calibrate_site_scale(st["u"])
    s_z = compute_scale(st["z"].channel_max, 8)
    s_xin = compute_scale(st["x_in"].channel_max, 8)
    out_w = w.out_proj
    if hadamard:
        b = d.had_block
        out_w = (had.fuse_hadamard_out_proj(out_w, di, 1, b) / np.float32(np.sqrt(b))).astype(np.float32)
    s_y = cal.calibrate_site_scale(st["y_had"]) if hadamard else compute_scale(st["r"].channel_max, 8)
    x_cell_scale = cmap.scales.reshape(-1)[cells].astype(np.float32)
    ssg = None
    if d.variant == "mamba2":
        gn = d.n_state_groups * d.d_state
        s_Bin = compute_scale(st["B_in"].channel_max, 8)
        s_Cin = compute_scale(st["C_in"].channel_max, 8)
        s_dt = compute_scale(st["dt"].channel_max, 8)
        ssg = cal.build_state_group_scales(st["B"], st["C"], d.n_state_groups, d.d_state,
                                           st["h"], cmap)
        in_out = np.concatenate([np.full(di, s_z), np.full(di, s_xin), np.full(gn, s_Bin), np.full(gn, s_Cin),
                                 np.full(d.n_heads, s_dt)]).astype(np.float32)
        conv_in = in_out[di:2 * di + 2 * gn].copy()
        conv_out = np.concatenate([x_cell_scale, np.repeat(ssg.scales_B, d.d_state),
                                   np.repeat(ssg.scales_C, d.d_state)]).astype(np.float32)
    else:
        in_out = np.concatenate([np.full(di, s_z), np.full(di, s_xin)]).astype(np.float32)
        conv_in = in_out[di:].copy()
        conv_out = x_cell_scale
        ssg = cal.build_state_group_scales(st["B"], st["C"], 1, d.d_state, st["h"], cmap)
    state_scale = ssg.scales_state.reshape(-1)[cells].astype(np.float32)
    g_in = _gemm_group(d.d_model)
    qb = QBlock(d, profile, make_qlinear(w.in_proj, kind, g_in), make_qlinear(out_w, kind, _gemm_group(di)),
                w.conv_weight, w.conv_bias, w.a_log, w.d_param, w.dt_bias, w.norm_weight, w.head_group,
                s_u=s_u, in_out_scale=in_out, conv_in_scale=conv_in, conv_out_scale=conv_out,
                state_scale=state_scale, s_y=s_y, hadamard=hadamard, extra=dict(extra, ssg=ssg))
    if d.variant == "mamba1":
        R, N = d.dt_rank, d.d_state
        xw = (w.x_proj * x_cell_scale[None, :]).astype(np.float32)     # fold clustered x scale
        qb.x_proj = make_qlinear(xw, kind, _gemm_group(di))
        s_dtl = compute_scale(st["dt_low"].channel_max, 8)
        s_B = compute_scale(st["B"].channel_max, 8)
        s_C = compute_scale(st["C"].channel_max, 8)
        qb.xproj_out_scale = np.concatenate([np.full(R, s_dtl), np.full(N, s_B), np.full(N, s_C)]).astype(np.float32)
        qb.dt_proj = make_qlinear(w.dt_proj, kind, _gemm_group(R))
        qb.s_dt = compute_scale(st["dt"].channel_max, 8)
    return qb


def cmd_quantize(model: FloatModel, tokens, profiles, m=4, n=4, hadamard=True, reorder=True, seed=0,
                 head_bits=4, emb_bits=8):
    """SPEC.md:588-596 over a whole model (profiles: one per block)."""
    if isinstance(profiles, str):
        profiles = [profiles] * len(model.blocks)
    stats = collect_stats(model, tokens)
    blocks = [quantize_block(b, stats[l], profiles[l], m, n, hadamard, reorder, seed)
              for l, b in enumerate(model.blocks)]
    es = np.array([compute_scale(model.embedding[v], emb_bits) for v in range(model.embedding.shape[0])], np.float32)
    ec = quantize_codes(model.embedding, es[:, None], emb_bits)
    head = make_qlinear(model.head, "w4a8" if head_bits == 4 else "w8", _gemm_group(model.dims.d_model))
    s_head = cal.calibrate_site_scale(stats[-1]["head_in"])
    return QuantModel(model.dims, list(profiles), ec, es, model.layer_norms, blocks, model.final_norm, head, s_head,
                      extra={"emb_bits": emb_bits})


def quant_forward(qm: QuantModel, tokens, states=None, trace=None):
    """Prefill one sequence: tokens [T] → (logits [T×V], states)."""
    h = (qm.emb_codes[np.asarray(tokens)].astype(np.float32) * qm.emb_scale[np.asarray(tokens)][:, None]).astype(np.float32)
    new_states = []
    for l, qb in enumerate(qm.blocks):
        u = rmsnorm(h, qm.layer_norms[l])
        st = states[l] if states is not None else None
        tr = {} if trace is not None else None
        out, s = block_forward_quantized(u, qb, st, trace=tr)
        if trace is not None:
            trace.append(tr)
        new_states.append(s)
        h = (h + out).astype(np.float32)
    hf = rmsnorm(h, qm.final_norm)
    hq = quantize_codes(hf, qm.s_head, 8)
    logits, _ = qlinear_a8(hq, qm.head, qm.s_head)
    return logits, new_states


def generate(qm: QuantModel, prompt, n_new: int):
    """Greedy generate (derived from SsmState stepping)."""
    logits, states = quant_forward(qm, prompt)
    out = []
    tok = int(np.argmax(logits[-1]))
    for _ in range(n_new):
        out.append(tok)
        logits, states = quant_forward(qm, [tok], states)
        tok = int(np.argmax(logits[-1]))
    return np.array(out)
