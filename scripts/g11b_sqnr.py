"""LEDGER G11b measurement: W4A8 weight-scale schemes on the toy model (CPU oracle).

Schemes (all 4-bit codes, group 128 along K):
  spec    per-group float scale s_g = max|w_g|/7 — per-group int32
          partials promoted to f32 (what the B200 GEMM now does)
  prog    round-1 progressive s_ch*sg, sg integer in [1,15], s_ch = max_g s_g / 15
  prog_nz progressive with s_ch taken over non-zero groups only (ADVICE r1 fix)
Reports weight SQNR and end-to-end logits SQNR vs the float model (dB)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pipeline as opl, qblock as qbm
from oracle.ssm_block import Dims
from oracle.quantizer import compute_scale, quantize_codes


def sqnr(ref, x):
    ref = np.asarray(ref, np.float64); x = np.asarray(x, np.float64)
    return 10 * np.log10((ref ** 2).sum() / max(((ref - x) ** 2).sum(), 1e-300))


def scales(w, scheme, group=128):
    n, k = w.shape
    wg = w.reshape(n, k // group, group)
    m = np.abs(wg).max(-1)
    s = np.where(m == 0, 1.0, m / 7).astype(np.float32)
    if scheme == "spec":
        return s
    if scheme == "prog":
        sch = (s.max(1) / 15).astype(np.float32)
    else:
        sch = (np.where(m == 0, 0, s).max(1) / 15).astype(np.float32)
        sch = np.where(sch == 0, np.float32(1 / 15), sch).astype(np.float32)
    sg = np.clip(np.ceil(s / sch[:, None]), 1, 15)
    return (sch[:, None] * sg).astype(np.float32)


def dequant(w, scheme, group=128):
    n, k = w.shape
    s = scales(w, scheme, group)
    q = quantize_codes(w.reshape(n, k // group, group), s[:, :, None], 4)
    return (q.astype(np.float32) * s[:, :, None]).reshape(n, k)


def main():
    d = Dims("mamba2", 256, 512, 64, 8, 64, 2, 4)
    fm = opl.cmd_gen_toy(d, 2, seed=0)
    toks = opl.calib_tokens(512, 4, 64)
    ev = opl.calib_tokens(512, 2, 64, seed=1)
    # weight-level SQNR over every block projection, plus a row with one all-zero group
    print("weight SQNR (dB)")
    for name, w in [("in_proj", fm.blocks[0].in_proj), ("out_proj", fm.blocks[0].out_proj), ("head", fm.head)]:
        print(f"  {name:9s}", "  ".join(f"{s}={sqnr(w, dequant(w, s)):.2f}" for s in ("spec", "prog", "prog_nz")))
    w = fm.blocks[0].in_proj.copy(); w[:, :128] = 0
    print("  zero-grp ", "  ".join(f"{s}={sqnr(w, dequant(w, s)):.2f}" for s in ("spec", "prog", "prog_nz")))
    # model-level: swap the float weights for each scheme's dequantised weights (W4 part only)
    ref = np.concatenate([opl.float_forward(fm, t) for t in ev])
    print("logits SQNR vs float model, weights-only 4-bit (dB)")
    for s in ("spec", "prog", "prog_nz"):
        fq = opl.cmd_gen_toy(d, 2, seed=0)
        for b in fq.blocks:
            b.in_proj = dequant(b.in_proj, s); b.out_proj = dequant(b.out_proj, s)
        fq.head = dequant(fq.head, s)
        out = np.concatenate([opl.float_forward(fq, t) for t in ev])
        print(f"  {s:8s} {sqnr(ref, out):.2f}")
    qm = opl.cmd_quantize(fm, toks, "W4A8")
    out = np.concatenate([opl.quant_forward(qm, t)[0] for t in ev])
    print(f"full W4A8 pipeline (oracle's current scheme): {sqnr(ref, out):.2f} dB")


if __name__ == "__main__":
    main()
