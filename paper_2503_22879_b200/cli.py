"""cli — SPEC `[MODULE] cli_pipeline`: toy-model generation and the
quantize pipeline (the kept entry points), plus the console script `ssmquant`
(pkg/pyproject.toml:16 declares `ssmquant.cli:main`).

gen-toy: weights N(0, 1/√fan_in); the x rows of in_proj carry per-channel
log-uniform multipliers spanning 100× (channel persistence, Fig. 3);
a_log = log U[1,16] (A < 0); dt_bias = softplus⁻¹(U[1e-3, 1e-1]); D = 1; Student-t(ν=3)
embedding rows with per-channel scales.  Every tensor draws from make_rng(seed, layer, id),
so the same seed gives the same model as the test oracle.

quantize, fixed stage order: collect_stats (float model, on the GPU) ->
sort_and_cluster -> build_state_group_scales -> reorder -> Hadamard fusion of out_proj (A8)
-> weight quantisation -> activation-scale embedding -> head-to-toe (per-row int8
embedding, W4A8 head).  The result feeds model.QuantizedMambaLM.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import sys
from dataclasses import dataclass, field

import numpy as np
import torch

from . import calibrate as cal
from . import hadamard as had
from . import reorder as ro
from .errors import PipelineError, SsmQuantError
from .quantizer import compute_scale, gptq_quantize_weight, quantize_weight_w4, quantize_weight_w4a8, quantize_weight_w8
from .ssm_block import Dims, QBlock, QLinear, SsmBlockWeights
from .tensor import make_rng

T_IN, T_CONV_W, T_CONV_B, T_ALOG, T_DTB, T_NORM, T_OUT, T_XPROJ, T_DTPROJ, T_MULT, T_BCG, T_NOUT = range(12)


def gen_block(d: Dims, seed: int, layer: int, n_layers: int = 1) -> SsmBlockWeights:
    r = lambda t: make_rng(seed, layer + 1, t)   # noqa: E731
    di, dm, K = d.d_inner, d.d_model, d.conv_kernel
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
    """SPEC.md:579-587 (returns the model; `main gen-toy` writes it as an archive)."""
    r = lambda t: make_rng(seed, 0, t)   # noqa: E731
    chs = np.exp(r(1).uniform(np.log(0.1), np.log(10.0), d.d_model))
    emb = (r(2).standard_t(3, (vocab, d.d_model)) * chs).astype(np.float32)
    lns = [(1.0 + 0.1 * make_rng(seed, 1000 + l, 0).standard_normal(d.d_model)).astype(np.float32)
           for l in range(n_blocks)]
    blocks = [gen_block(d, seed, l, n_blocks) for l in range(n_blocks)]
    head = (r(3).standard_normal((vocab, d.d_model)) / np.sqrt(d.d_model)).astype(np.float32)
    return FloatModel(d, emb, lns, blocks, np.ones(d.d_model, np.float32), head)


def calib_tokens(vocab: int, n_samples: int, seq_len: int, seed: int = 0) -> np.ndarray:
    return make_rng(seed, 7, 7).integers(0, vocab, (n_samples, seq_len))


def _gemm_group(k: int) -> int:
    return 128 if k % 128 == 0 else (32 if k % 32 == 0 else k)


def make_qlinear(w, kind: str, group: int = 128, calib=None) -> QLinear:
    """``calib`` (rows of this projection's input, in the weight's column basis) switches the
    4-bit kinds from round-to-nearest to GPTQ (the Table 7 "GPTQ" toggle)."""
    w = np.asarray(w, np.float32)
    group = min(group, w.shape[1])
    n = lambda t: t.cpu().numpy()   # noqa: E731
    if kind == "w8":
        q = quantize_weight_w8(w)
        return QLinear("w8", n(q.payload), s_ch=n(q.extra["s_ch"]), group=w.shape[1])
    if kind in ("w4a8", "w4a16"):
        if calib is not None:
            q = gptq_quantize_weight(w, calib, 4, group, device=getattr(calib, "device", None))
        else:
            q = quantize_weight_w4a8(w, group) if kind == "w4a8" else quantize_weight_w4(w, group)
        return QLinear(kind, n(q.payload), s_group=n(q.extra["s_group"]), group=group)
    raise PipelineError(f"unknown weight kind {kind}")


@dataclass
class QuantModel:
    """Head-to-toe quantized model (consumed by model.QuantizedMambaLM)."""
    dims: Dims
    profiles: list
    emb_codes: np.ndarray
    emb_scale: np.ndarray
    layer_norms: list
    blocks: list
    final_norm: np.ndarray
    head: QLinear
    s_head: np.float32
    extra: dict = field(default_factory=dict)


def quantize_block(blk: SsmBlockWeights, st: dict, profile: str, m=4, n=4, hadamard=True, reorder=True, seed=0,
                   gptq=False, persg=True, snc=True):
    """SPEC.md:591 stages for one block from its calibration stats.  ``gptq`` (4-bit profiles):
    the projections are rounded by GPTQ on the calibration rows kept by collect_stats(keep_rows),
    each mapped into its weight's column basis (reordered, Hadamard-rotated, cluster-scaled).
    Table 7 ablation toggles: ``persg=False`` gives B / C one per-tensor scale
    each instead of per-state-group scales, ``snc=False`` one x scale (m = n = 1) instead of the
    sort-and-cluster cells."""
    d = blk.dims
    di = d.d_inner
    nh, P = (d.n_heads, d.head_dim) if d.variant == "mamba2" else (1, d.d_inner)
    if not snc:
        m = n = 1
    cmap = cal.sort_and_cluster(st["x"], nh, P, m, n, seed)
    plan = ro.build_reorder_plan(cmap, d)
    w = ro.apply_reorder(blk, plan) if reorder else blk
    cells = cmap.cell_of_new()
    if not reorder:                      # clustered scales looked up in the original layout
        c0 = np.empty_like(cells)
        c0[plan.pi] = cells
        cells = c0
    kind = {"W8A8": "w8", "W4A8": "w4a8", "W4A16": "w4a16"}[profile]
    extra = {"cmap": cmap, "plan": plan}
    rows = st.get("_rows") if (gptq and kind != "w8") else None
    if gptq and kind != "w8" and not rows:
        raise PipelineError("gptq needs calibration rows: collect_stats(..., keep_rows=N)")
    pi = plan.pi if reorder else np.arange(di)
    cal_in = rows["u"].float() if rows else None                           # in_proj input
    cal_dtl = rows["dt_low"].float() if rows and "dt_low" in rows else None   # Mamba1 dt_proj input
    cal_r = rows["r"].float()[:, torch.as_tensor(pi, device=rows["r"].device)] if rows else None
    cal_x = rows["x"].float()[:, torch.as_tensor(pi, device=rows["x"].device)] if rows and d.variant == "mamba1" else None
    if profile == "W4A16":
        qb = QBlock(d, profile, make_qlinear(w.in_proj, kind, _gemm_group(d.d_model), cal_in),
                    make_qlinear(w.out_proj, kind, _gemm_group(di), cal_r), w.conv_weight, w.conv_bias, w.a_log,
                    w.d_param, w.dt_bias, w.norm_weight, w.head_group, extra=extra)
        if d.variant == "mamba1":
            qb.x_proj = make_qlinear(w.x_proj, kind, _gemm_group(di), cal_x)
            qb.dt_proj = make_qlinear(w.dt_proj, kind, _gemm_group(d.dt_rank), cal_dtl)
        return qb
    s_u = cal.calibrate_site_scale(st["u"])
    s_z = compute_scale(st["z"].channel_max, 8)
    s_xin = compute_scale(st["x_in"].channel_max, 8)
    out_w = w.out_proj
    if hadamard:
        b = d.had_block
        out_w = (had.fuse_hadamard_out_proj(out_w, di, 1, b).numpy() / np.float32(np.sqrt(b))).astype(np.float32)
    s_y = cal.calibrate_site_scale(st["y_had"]) if hadamard else compute_scale(st["r"].channel_max, 8)
    x_cell_scale = cmap.scales.reshape(-1)[cells].astype(np.float32)
    if d.variant == "mamba2":
        gn = d.n_state_groups * d.d_state
        s_Bin, s_Cin = compute_scale(st["B_in"].channel_max, 8), compute_scale(st["C_in"].channel_max, 8)
        s_dt = compute_scale(st["dt"].channel_max, 8)
        ssg = cal.build_state_group_scales(st["B"], st["C"], d.n_state_groups, d.d_state, st["h"], cmap)
        if not persg:   # one B and one C scale over every state group
            ssg = dataclasses.replace(ssg, scales_B=np.full_like(ssg.scales_B, ssg.scales_B.max()),
                                      scales_C=np.full_like(ssg.scales_C, ssg.scales_C.max()))
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
    if cal_r is not None and hadamard:   # out_proj sees the unnormalised blocked FWHT of r
        cal_r = had.fwht_blocked(cal_r, d.had_block)
    qb = QBlock(d, profile, make_qlinear(w.in_proj, kind, _gemm_group(d.d_model), cal_in),
                make_qlinear(out_w, kind, _gemm_group(di), cal_r), w.conv_weight, w.conv_bias, w.a_log, w.d_param,
                w.dt_bias, w.norm_weight, w.head_group, s_u=s_u, in_out_scale=in_out, conv_in_scale=conv_in,
                conv_out_scale=conv_out, state_scale=state_scale, s_y=s_y, hadamard=hadamard,
                extra=dict(extra, ssg=ssg))
    if d.variant == "mamba1":
        R, N = d.dt_rank, d.d_state
        if cal_x is not None:   # x_proj's GEMM input is x / (clustered x scale)
            cal_x = cal_x / torch.as_tensor(x_cell_scale, device=cal_x.device)[None, :]
        qb.x_proj = make_qlinear((w.x_proj * x_cell_scale[None, :]).astype(np.float32), kind, _gemm_group(di), cal_x)
        s_dtl = compute_scale(st["dt_low"].channel_max, 8)
        qb.xproj_out_scale = np.concatenate([np.full(R, s_dtl), np.full(N, compute_scale(st["B"].channel_max, 8)),
                                             np.full(N, compute_scale(st["C"].channel_max, 8))]).astype(np.float32)
        qb.dt_proj = make_qlinear(w.dt_proj, kind, _gemm_group(R), cal_dtl)
        qb.s_dt = compute_scale(st["dt"].channel_max, 8)
    return qb


def cmd_quantize(model: FloatModel, tokens, profiles, m=4, n=4, hadamard=True, reorder=True, seed=0,
                 head_bits=4, emb_bits=8, device="cuda", stats=None, gptq=False, gptq_rows=512) -> QuantModel:
    """SPEC.md:588-596 over a whole model (``profiles``: one per block or a single name).
    ``gptq``: 4-bit projections by GPTQ on ``gptq_rows`` calibration rows per projection."""
    if isinstance(profiles, str):
        profiles = [profiles] * len(model.blocks)
    if len(profiles) != len(model.blocks):
        raise PipelineError("one profile per block")
    stats = stats if stats is not None else cal.collect_stats(model, tokens, device=device,
                                                               keep_rows=gptq_rows if gptq else 0)
    blocks = [quantize_block(b, stats[l], profiles[l], m, n, hadamard, reorder, seed, gptq)
              for l, b in enumerate(model.blocks)]
    emb = np.asarray(model.embedding, np.float32)
    es = np.array([compute_scale(emb[v], emb_bits) for v in range(emb.shape[0])], np.float32)
    lo, hi = -(1 << (emb_bits - 1)), (1 << (emb_bits - 1)) - 1
    ec = np.clip(np.rint(emb / es[:, None]), lo, hi).astype(np.int8)
    head = make_qlinear(model.head, "w4a8" if head_bits == 4 else "w8", _gemm_group(model.dims.d_model))
    return QuantModel(model.dims, list(profiles), ec, es, model.layer_norms, blocks, model.final_norm, head,
                      cal.calibrate_site_scale(stats[-1]["head_in"]), extra={"emb_bits": emb_bits})


# ------------------------------------------------------------------ console script
def main(argv=None) -> int:
    """`ssmquant gen-toy | quantize | inspect`; any SsmQuantError -> exit 1."""
    ap = argparse.ArgumentParser(prog="ssmquant")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen-toy")
    g.add_argument("--dims", default="mamba2,256,512,64,8,64,2,4")
    g.add_argument("--blocks", type=int, default=2)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--vocab", type=int, default=512)
    g.add_argument("--out", required=True)
    q = sub.add_parser("quantize")
    q.add_argument("--model", required=True)
    q.add_argument("--profile", default="W8A8", choices=["W8A8", "W4A8", "W4A16"])
    q.add_argument("--samples", type=int, default=8)
    q.add_argument("--seq-len", type=int, default=64)
    q.add_argument("--no-hadamard", action="store_true")
    q.add_argument("--no-reorder", action="store_true")
    q.add_argument("--gptq", action="store_true", help="GPTQ for the 4-bit projections (SPEC.md:146)")
    q.add_argument("--out", required=True)
    i = sub.add_parser("inspect")
    i.add_argument("archive")
    a = ap.parse_args(argv)
    try:
        from . import archive
        if a.cmd == "gen-toy":
            f = a.dims.split(",")
            d = Dims(f[0], *[int(v) for v in f[1:]])
            fm = cmd_gen_toy(d, a.blocks, a.seed, a.vocab)
            archive.write_float_model(fm, a.out)
        elif a.cmd == "quantize":
            fm = archive.read_float_model(a.model)
            toks = calib_tokens(fm.embedding.shape[0], a.samples, a.seq_len)
            import torch
            dev = "cuda" if torch.cuda.is_available() else "cpu"   # offline calibration forward
            qm = cmd_quantize(fm, toks, a.profile, hadamard=not a.no_hadamard, reorder=not a.no_reorder, device=dev,
                              gptq=a.gptq)
            archive.write_quant_model(qm, a.out)
        else:
            print(json.dumps(archive.inspect(a.archive), indent=1))
    except SsmQuantError as e:
        print(f"ssmquant: {type(e).__name__}: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
