"""Benchmark of the quantized Mamba block hot path on B200 (driver contract: one JSON line).

Default workload (BASELINE.json `metric`, configs[2]): Mamba2-8B-shaped W4A8 decode,
batch 64 per GPU, 56 layers + W4A8 head + greedy argmax, int8 SSM state — one step =
one token for every sequence, replayed from a CUDA graph.  Inputs per step (weights
3.3 GB + int8 state 7.5 GB) are far larger than L2, so no L2 flush is needed.

    python bench.py [--gpus N --steps K --warmup W] [--workload decode8b|prefill27b|decode8b_w4a16]
    python bench.py --impl reference      # CPU reference arm (oracle port on host cores)

Multi-GPU (torchrun): batch-sharded replicas, no collective on the path; every rank runs
its own 64 sequences (weak scaling); timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0
FALLBACK_BF16 = 1590.0

WORKLOADS = {
    "decode8b": dict(dims=("mamba2", 4096, 8192, 128, 128, 64, 8, 4), layers=56, vocab=256000, profile="W4A8",
                     batch=64, desc="Mamba2-8B-shaped W4A8 decode, batch 64/GPU, int8 state, 56 layers + W4A8 head"),
    "prefill27b": dict(dims=("mamba2", 2560, 5120, 128, 80, 64, 1, 4), layers=64, vocab=50288, profile="W8A8",
                       batch=8, seq=2048,
                       desc="Mamba2-2.7B-shaped W8A8 prefill, batch 8 x 2048 tokens/GPU, 64 layers, last-token head"),
    "decode8b_w4a16": dict(dims=("mamba2", 4096, 8192, 128, 128, 64, 8, 4), layers=56, vocab=256000,
                           profile="W4A16", batch=1,
                           desc="Mamba2-8B-shaped W4A16 decode, batch 1, fp32 state, 56 layers + W4A8 head"),
    # configs[4]: Mamba1-2.8B W8A8, the paper's TTFT protocol (b=1, 1024-token prefill) and decode
    "m1prefill28b": dict(dims=("mamba1", 2560, 5120, 16, 1, 5120, 1, 4, 160), layers=64, vocab=50288,
                         profile="W8A8", batch=1, seq=1024, model="Mamba1-2.8B-shaped",
                         desc="Mamba1-2.8B-shaped W8A8 prefill, batch 1 x 1024 tokens, 64 layers, last-token head"),
    "m1decode28b": dict(dims=("mamba1", 2560, 5120, 16, 1, 5120, 1, 4, 160), layers=64, vocab=50288,
                        profile="W8A8", batch=1, model="Mamba1-2.8B-shaped",
                        desc="Mamba1-2.8B-shaped W8A8 decode, batch 1, int8 state, 64 layers + W4A8 head"),
}


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return FALLBACK_HBM, FALLBACK_BF16, "fallback"


_INT8_PEAK = None


def int8_peak_tops(dev) -> float:
    """Dense INT8 tensor peak measured here: torch._int_mm (cuBLASLt) on 8192^3, best of 10
    (the driver's MEASURED_PEAKS.json has no INT8 figure)."""
    global _INT8_PEAK
    if _INT8_PEAK is None:
        import torch
        n = 8192
        a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device=dev)
        b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device=dev).t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        _INT8_PEAK = 2.0 * n ** 3 / best / 1e12
        del a, b
    return _INT8_PEAK


class Clocks:
    """Samples nvidia-smi clocks/throttle reasons during the timed region."""

    def __init__(self, idx):
        self.idx = idx
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(kernel_name, pattern=None):
    """dram read+write bytes per launch of `kernel_name` from the newest committed ncu --set full
    summary (profiles/*.txt written by scripts/summarize_profiles.py), or None.  For the decode SSM
    step (prep_kernel + state_ring_kernel + norm_had8192_kernel) the three kernels' bytes are summed."""
    import glob
    import re
    step = kernel_name.startswith("mamba2_decode_step_int8")
    if pattern is None:
        pattern = "*prof_ring*.txt" if step or kernel_name.startswith("state_ring") else "*prof_prefill*.txt"
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", pattern)))
    if not files:
        return None
    txt = open(files[-1]).read()
    keys = ("prep_kernel", "state_ring_kernel", "norm_had8192_kernel") if step else (kernel_name.split()[0],)
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total = 0.0
    for key in keys:
        ids = [m.group(1) for m in re.finditer(r"## ID (\d+): (?:void )?(\S+)", txt) if m.group(2).startswith(key)]
        if not ids:
            return None
        m = re.search(r"## raw ID %s: dram__bytes_read.sum=([0-9.]+) (\w+); dram__bytes_write.sum=([0-9.]+) (\w+)"
                      % ids[0], txt)
        if not m:
            return None
        total += float(m.group(1)) * unit.get(m.group(2), 1) + float(m.group(3)) * unit.get(m.group(4), 1)
    return total


def dist_init():
    from paper_2503_22879_b200 import dist as pdist
    return pdist.init("nccl")


def max_over_ranks(v, world):
    from paper_2503_22879_b200 import dist as pdist
    return pdist.max_over_ranks(v, world)


def barrier(world):
    from paper_2503_22879_b200 import dist as pdist
    pdist.barrier(world)


# ------------------------------------------------------------------ CPU baseline (oracle)
def cpu_decode_sample(dims, profile, batch, layers_sample=2, seed=0):
    """Time the oracle (numpy port) on a bounded sample: `layers_sample` full-width layers of
    one decode step at the full batch, extrapolated to the model's layer count."""
    from oracle import qblock as oq
    from oracle.ssm_block import Dims as ODims
    from paper_2503_22879_b200 import synth
    from paper_2503_22879_b200.ssm_block import Dims
    d = Dims(*dims)
    od = ODims(*dims)
    qb = synth.random_qblock(d, profile, seed)
    qb.dims = od
    oqb = oq.QBlock(od, qb.profile, oq.QLinear(**vars(qb.in_proj)), oq.QLinear(**vars(qb.out_proj)),
                    qb.conv_weight, qb.conv_bias, qb.a_log, qb.d_param, qb.dt_bias, qb.norm_weight, qb.head_group,
                    s_u=qb.s_u, in_out_scale=qb.in_out_scale, conv_in_scale=qb.conv_in_scale,
                    conv_out_scale=qb.conv_out_scale, state_scale=qb.state_scale, s_y=qb.s_y)
    r = np.random.default_rng(seed)
    u = r.standard_normal((batch, d.d_model)).astype(np.float32)
    h = r.integers(-100, 100, (batch, d.n_heads, d.head_dim, d.d_state)).astype(np.int8)
    c = r.integers(-100, 100, (batch, d.conv_dim, d.conv_kernel - 1)).astype(np.int8)
    t0 = time.perf_counter()
    for _ in range(layers_sample):
        out, h, c = oq.decode_step_batched(u, oqb, h, c)
    dt = (time.perf_counter() - t0) / layers_sample
    return dt


def _oracle_qblock(qb, od):
    """The oracle's QBlock for a synthetic product QBlock (Mamba2 or Mamba1 fields)."""
    from oracle import qblock as oq
    ql = lambda q: None if q is None else oq.QLinear(**vars(q))   # noqa: E731
    return oq.QBlock(od, qb.profile, ql(qb.in_proj), ql(qb.out_proj), qb.conv_weight, qb.conv_bias, qb.a_log,
                     qb.d_param, qb.dt_bias, qb.norm_weight, qb.head_group, x_proj=ql(getattr(qb, "x_proj", None)),
                     dt_proj=ql(getattr(qb, "dt_proj", None)), s_u=qb.s_u, in_out_scale=qb.in_out_scale,
                     conv_in_scale=qb.conv_in_scale, conv_out_scale=qb.conv_out_scale, state_scale=qb.state_scale,
                     s_y=qb.s_y, xproj_out_scale=getattr(qb, "xproj_out_scale", None), s_dt=getattr(qb, "s_dt", 1.0))


def cpu_prefill_sample(dims, profile, tokens, seed=0):
    """Time the oracle (numpy port) prefill of one full-width layer over `tokens` tokens of one
    sequence (chunked SSD path); returns seconds per token per layer."""
    from oracle import qblock as oq
    from oracle.ssm_block import Dims as ODims
    from paper_2503_22879_b200 import synth
    from paper_2503_22879_b200.ssm_block import Dims
    d = Dims(*dims)
    od = ODims(*dims)
    qb = synth.random_qblock(d, profile, seed)
    oqb = _oracle_qblock(qb, od)
    u = np.random.default_rng(seed).standard_normal((tokens, d.d_model)).astype(np.float32)
    t0 = time.perf_counter()
    oq.block_forward_quantized(u, oqb)
    return (time.perf_counter() - t0) / tokens


def run_reference_arm(args, wl, world, rank):
    if rank != 0:
        return
    import multiprocessing
    cores = multiprocessing.cpu_count()
    if "seq" in wl:   # prefill workloads
        ntok = 128
        cpu_prefill_sample(wl["dims"], wl["profile"], 16)
        spts = [cpu_prefill_sample(wl["dims"], wl["profile"], ntok) for _ in range(args.steps)]
        val = 1.0 / (float(np.mean(spts)) * wl["layers"])
        line = {"impl": "reference", "metric": "prefill tok/s", "value": val, "unit": "tok/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wl["batch"] * wl["seq"] / val,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
                "data": "synthetic", "config": {"workload": args.workload, "desc": wl["desc"]},
                "cpu_baseline": {"value": val, "unit": "tok/s", "cores": cores, "kind": "port",
                                 "sample": f"one full-width layer over {ntok} tokens per timed step, x{wl['layers']} "
                                           f"layers (extrapolated); numpy oracle, exact-int f64 BLAS"},
                "e2e": {"value": val, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    b = wl["batch"] * world
    per_layer = []
    for _ in range(max(1, args.warmup and 1)):
        cpu_decode_sample(wl["dims"], wl["profile"], wl["batch"], 1)
    for _ in range(args.steps):
        per_layer.append(cpu_decode_sample(wl["dims"], wl["profile"], wl["batch"], 1))
    step_s = float(np.mean(per_layer)) * wl["layers"]
    val = wl["batch"] / step_s
    line = {"impl": "reference", "metric": "decode tok/s", "value": val, "unit": "tok/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
            "config": {"workload": args.workload, "desc": wl["desc"]},
            "cpu_baseline": {"value": val, "unit": "tok/s", "cores": cores, "kind": "port",
                             "sample": f"1 full-width layer of one b={wl['batch']} decode step per timed step, "
                                       f"x{wl['layers']} layers (extrapolated); numpy oracle, exact-int f64 BLAS"},
            "e2e": {"value": val, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_prefill(args, wl, world, rank, local, emit=True):
    """configs[1]: one step = prefill of batch x seq tokens through every layer (fresh state,
    int8 final state written), last-token logits; tokens from pinned host memory for e2e.
    Returns the line (rank 0); prints it when ``emit``."""
    import torch
    from paper_2503_22879_b200 import ops, synth
    from paper_2503_22879_b200.ssm_block import Dims
    import __graft_entry__
    __graft_entry__.build()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    d = Dims(*wl["dims"])
    B, T = wl["batch"], wl["seq"]
    lm = synth.synthetic_lm(d, wl["layers"], wl["profile"], wl["vocab"], dev, seed=rank)
    states = lm.new_states(B)
    ws = lm._workspace(B * T)
    g = torch.Generator(device=dev)
    g.manual_seed(11 + rank)
    tok = torch.randint(0, wl["vocab"], (B * T,), generator=g, device=dev, dtype=torch.int32)

    def step():
        return lm._run(tok, B, T, states, False, ws, False)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        e0.record(st)
        for _ in range(args.steps):
            step()
        e1.record(st)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    value = world * B * T / (ms / 1e3)
    pin_in = torch.randint(0, wl["vocab"], (B * T,), dtype=torch.int32).pin_memory()
    pin_out = torch.empty((B, lm.vocab), dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(st)
    for _ in range(args.steps):
        tok.copy_(pin_in, non_blocking=True)
        lg = step()
        pin_out.copy_(lg, non_blocking=True)
        st.synchronize()
    t1.record(st)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(t0.elapsed_time(t1) / args.steps, world)
    # dominant op: the in_proj W8A8 GEMM (int8 tensor cores), timed live on its stream
    blk = lm.blocks[0]
    M = B * T
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        blk.in_proj.a8(ws["u"], ops.EPI_QUANT, ws["zx"], blk.in_out_scale)
    torch.cuda.synchronize()
    reps = 10
    k0.record(st)
    for i in range(reps):
        lm.blocks[i % len(lm.blocks)].in_proj.a8(ws["u"], ops.EPI_QUANT, ws["zx"], blk.in_out_scale)
    k1.record(st)
    torch.cuda.synchronize()
    gemm_ms = k0.elapsed_time(k1) / reps
    ops_per = 2.0 * M * d.in_proj_out * d.d_model
    achieved = ops_per / (gemm_ms / 1e3) / 1e12
    hbm, bf16, pk_kind = peaks()
    i8peak = int8_peak_tops(dev)
    # the step's largest kernel: the chunked int8 SSD scan (HBM-bound in principle: int8 codes
    # in, f32 y + int8 state out), timed live on the layer's own inputs (Mamba2); Mamba1's
    # largest kernel is the in_proj GEMM itself
    launches_per_step = ops.LAUNCH_COUNTER[0]
    ops.LAUNCH_COUNTER[0] = 0
    step()
    torch.cuda.synchronize()
    launches_per_step, ops.LAUNCH_COUNTER[0] = ops.LAUNCH_COUNTER[0], launches_per_step
    if d.variant == "mamba1":
        return _prefill_line(args, wl, world, rank, d, B, T, value, ms, e2e_ms, lm, clk, achieved, i8peak, pk_kind,
                             ops_per, gemm_ms, launches_per_step, emit)
    di, gn, nh = d.d_inner, d.n_state_groups * d.d_state, d.n_heads
    cv, zx = ws["conv"], ws["zx"]
    st_tmp = torch.empty((B, nh, d.head_dim, d.d_state), dtype=torch.int8, device=dev)

    def ssd():
        ops.ssd_scan_int8(blk.params, B, T, cv[:, :di], cv[:, di:di + gn], cv[:, di + gn:], zx[:, 2 * di + 2 * gn:],
                          zx[:, :di], st_tmp, False, ws["y"])
    for _ in range(2):
        ssd()
    torch.cuda.synchronize()
    k0.record(st)
    for _ in range(5):
        ssd()
    k1.record(st)
    torch.cuda.synchronize()
    ssd_ms = k0.elapsed_time(k1) / 5
    ssd_bytes = M * (di + 2 * gn + di + nh + 4 * di) + st_tmp.numel()
    ssd_gbs = ssd_bytes / (ssd_ms / 1e3) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import multiprocessing
        ntok = 256
        spt = cpu_prefill_sample(wl["dims"], wl["profile"], ntok)
        cpu = {"value": 1.0 / (spt * wl["layers"]), "unit": "tok/s", "cores": multiprocessing.cpu_count(),
               "kind": "port", "sample": f"one full-width layer over {ntok} tokens of one sequence (chunked SSD), "
                                         f"x{wl['layers']} layers (extrapolated); numpy oracle, exact-int f64 BLAS"}
    if rank == 0:
        line = {"metric": "prefill tok/s", "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "int8", "data": "synthetic",
                "config": {"workload": wl.get("name", args.workload), "desc": wl["desc"], "model": "Mamba2-2.7B-shaped",
                           "global_batch": B * world, "seq_len": T, "layers": wl["layers"],
                           "parallelism": f"dp{world} (batch-shard replicas, no collective)",
                           "l2": "activations 16384 x 10576 int8 per layer exceed L2; no flush"},
                "roofline": {"bound": "hbm", "kernel": "ssd_chunk_kernel (chunked int8 SSD scan, mma.sync)",
                             "achieved": ssd_gbs, "peak": hbm, "unit": "GB/s", "frac": ssd_gbs / hbm,
                             "traffic": ncu_traffic("ssd_chunk_kernel<128>"), "peak_kind": pk_kind,
                             "algorithmic_bytes_per_launch": ssd_bytes, "launch_ms": ssd_ms},
                "roofline_gemm": {"bound": "tensor", "kernel": "gemm_tc_kernel (in_proj W8A8, tcgen05 kind::i8)",
                                  "achieved": achieved, "peak": i8peak, "unit": "TOP/s", "frac": achieved / i8peak,
                                  "traffic": None,
                                  "peak_kind": "measured here: torch._int_mm int8 8192^3 dense (cuBLASLt), best of 10",
                                  "algorithmic_ops_per_launch": ops_per, "launch_ms": gemm_ms},
                "cpu_baseline": cpu,
                "e2e": {"value": world * B * T / (e2e_ms / 1e3), "unit": "tok/s", "h2d_bytes_per_step": B * T * 4,
                        "d2h_bytes_per_step": B * lm.vocab * 4},
                "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary()}
        if emit:
            print(json.dumps(line), flush=True)
        return line
    return None


def _prefill_line(args, wl, world, rank, d, B, T, value, ms, e2e_ms, lm, clk, achieved, i8peak, pk_kind, ops_per,
                  gemm_ms, launches_per_step, emit=True):
    """Mamba1 prefill line: the in_proj W8A8 GEMM is the dominant kernel."""
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import multiprocessing
        ntok = 128
        spt = cpu_prefill_sample(wl["dims"], wl["profile"], ntok)
        cpu = {"value": 1.0 / (spt * wl["layers"]), "unit": "tok/s", "cores": multiprocessing.cpu_count(),
               "kind": "port", "sample": f"one full-width layer over {ntok} tokens of one sequence, "
                                         f"x{wl['layers']} layers (extrapolated); numpy oracle, exact-int f64 BLAS"}
    if rank == 0:
        line = {"metric": "prefill tok/s", "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "int8", "data": "synthetic",
                "config": {"workload": args.workload, "desc": wl["desc"], "model": wl.get("model", ""),
                           "global_batch": B * world, "seq_len": T, "layers": wl["layers"],
                           "parallelism": f"dp{world} (batch-shard replicas, no collective)"},
                "roofline": {"bound": "tensor", "kernel": "gemm_tc_kernel (in_proj W8A8, tcgen05 kind::i8)",
                             "achieved": achieved, "peak": i8peak, "unit": "TOP/s", "frac": achieved / i8peak,
                             "traffic": None,
                             "peak_kind": "measured here: torch._int_mm int8 8192^3 dense (cuBLASLt), best of 10",
                             "algorithmic_ops_per_launch": ops_per, "launch_ms": gemm_ms},
                "cpu_baseline": cpu,
                "e2e": {"value": world * B * T / (e2e_ms / 1e3), "unit": "tok/s", "h2d_bytes_per_step": B * T * 4,
                        "d2h_bytes_per_step": B * lm.vocab * 4},
                "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary()}
        if emit:
            print(json.dumps(line), flush=True)
        return line
    return None


def run_decode(args, wl, world, rank, local):
    import torch
    from paper_2503_22879_b200 import ops, synth
    from paper_2503_22879_b200.ssm_block import Dims
    import __graft_entry__
    __graft_entry__.build()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    d = Dims(*wl["dims"])
    from paper_2503_22879_b200 import dist as pdist
    tp_group = None
    if args.parallel == "heads":   # head shard: every rank runs the whole batch on nh/W heads per layer
        if d.variant != "mamba2":
            raise SystemExit("--parallel heads needs a Mamba2 workload")
        B = args.global_batch or wl["batch"]
        global_batch, scaling = B, "strong"
        if world > 1:
            import torch.distributed as tdist
            tp_group = tdist.group.WORLD
        parallelism = f"tp{world} (head shards, one NCCL all_reduce of the out_proj partials per layer)"
    elif args.global_batch:   # strong scaling: a fixed global batch sharded over the ranks
        lo, hi = pdist.shard_range(args.global_batch, world, rank)
        B = hi - lo
        global_batch, scaling = args.global_batch, "strong"
        parallelism = f"dp{world} (batch-shard replicas, no collective)"
    else:                   # weak scaling: wl["batch"] sequences per GPU
        B = wl["batch"]
        global_batch, scaling = B * world, "weak"
        parallelism = f"dp{world} (batch-shard replicas, no collective)"
    lm = synth.synthetic_lm(d, wl["layers"], wl["profile"], wl["vocab"], dev, seed=rank, tp_group=tp_group)
    states = lm.new_states(B)
    g = torch.Generator(device=dev)
    g.manual_seed(7 + rank)
    for s in states:    # start from a non-trivial cached state (decode after a prefill)
        if s.h.dtype == torch.int8:
            s.h.copy_(torch.randint(-100, 100, s.h.shape, generator=g, device=dev, dtype=torch.int8))
            s.conv_cache.copy_(torch.randint(-100, 100, s.conv_cache.shape, generator=g, device=dev,
                                             dtype=torch.int8))
        else:
            s.h.normal_(0, 0.1, generator=g)
    graph, tok, logits, ws = lm.capture_decode(B, states)
    launches_per_step = ops.LAUNCH_COUNTER[1]
    tok.copy_(torch.randint(0, wl["vocab"], (B,), generator=g, device=dev, dtype=torch.int32))
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    barrier(world)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.profiler.start()     # ncu --profile-from-start off captures exactly the timed steps
        e0.record(st)
        for _ in range(args.steps):
            graph.replay()
        e1.record(st)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    barrier(world)
    ms = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms, world)
    value = global_batch / (ms / 1e3)

    # e2e: host tokens in (pinned H2D), step, host tokens out (D2H) every step
    pin_in = torch.randint(0, wl["vocab"], (B,), dtype=torch.int32).pin_memory()
    pin_out = torch.empty(B, dtype=torch.int32).pin_memory()
    torch.cuda.synchronize()
    barrier(world)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(st)
    for _ in range(args.steps):
        tok.copy_(pin_in, non_blocking=True)
        graph.replay()
        pin_out.copy_(tok, non_blocking=True)
        st.synchronize()
        pin_in.copy_(pin_out)
    t1.record(st)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(t0.elapsed_time(t1) / args.steps, world)

    # dominant kernel class: the int8 SSM half of the decode step (K5d conv update, K9 state update,
    # K6 gated norm + FWHT + quant), timed live with CUDA events on the launch stream, cycling
    # through all layers' states (67 MB each at b=64, so every launch streams from HBM, not L2)
    blk = lm.blocks[0]
    d = blk.dims   # the blocks' dims (a head shard's under --parallel heads)
    di, gn = d.d_inner, d.n_state_groups * d.d_state
    reps = 2 * len(lm.blocks)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if d.variant == "mamba1":
        dom_name = "gemm_tc_kernel / gemm_a8_mma (in_proj W8A8, decode weight stream)"

        def dom(i):
            b_ = lm.blocks[i % len(lm.blocks)]
            b_.in_proj.a8(ws["u"][:B], ops.EPI_QUANT, ws["zx"][:B], b_.in_out_scale)
        dom_bytes = d.in_proj_out * d.d_model + B * (d.d_model + d.in_proj_out)
    elif blk.a8 and getattr(blk, "fused_decode", False):
        dom_name = "mamba2_decode_step_int8 (prep_kernel + state_ring_kernel + norm_had8192_kernel, decode)"

        def dom(i):
            b_ = lm.blocks[i % len(lm.blocks)]
            s_ = states[i % len(states)]
            ops.mamba2_decode_step_int8(b_.decode_params, B, ws["zx"], s_.conv_cache, s_.h, ws["yq"], ws["y"],
                                        ws["dws"])
        # strictly algorithmic bytes (no workspace): int8 state read + write, int8 conv cache read +
        # write, the in_proj codes read (z|x|B|C|dt), the int8 out_proj input written
        dom_bytes = (2 * B * d.n_heads * d.head_dim * d.d_state
                     + 2 * B * (d.conv_kernel - 1) * d.conv_dim
                     + B * d.in_proj_out + B * di)
    else:
        # W4A16: the in_proj GEMV streams the most bytes of the step (42% of the launch list)
        dom_name = "gemv_w4a16_mma_kernel (in_proj W4A16, decode weight stream)"

        def dom(i):
            b_ = lm.blocks[i % len(lm.blocks)]
            b_.in_proj.a16(ws["uf"][:B], ws["zxf"][:B])
        n_out = d.in_proj_out
        dom_bytes = n_out * d.d_model // 2 + n_out * (d.d_model // 128) * 4 + B * (d.d_model + n_out) * 4
    for i in range(5):
        dom(i)
    torch.cuda.synchronize()
    k0.record(st)
    for i in range(reps):
        dom(i)
    k1.record(st)
    torch.cuda.synchronize()
    dom_ms = k0.elapsed_time(k1) / reps
    hbm, bf16, pk_kind = peaks()
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9

    step_bytes = lm.weight_bytes() + sum(s.h.numel() * s.h.element_size() * 2 +
                                         s.conv_cache.numel() * s.conv_cache.element_size() * 2 for s in states)
    res = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        t = (cpu_decode_sample(wl["dims"], wl["profile"], B, layers_sample=2)
             if blk.a8 and d.variant == "mamba2" else None)
        if t is not None:
            import multiprocessing
            res = {"value": B / (t * wl["layers"]), "unit": "tok/s", "cores": multiprocessing.cpu_count(),
                   "kind": "port",
                   "sample": f"2 full-width layers of one b={B} decode step, x{wl['layers']} layers (extrapolated); "
                             "numpy oracle with exact-int f64 BLAS on all host threads"}
    prefill = None
    if args.workload == "decode8b" and not args.no_prefill:
        # configs[1] (the metric's prefill half) measured in the same run on a Mamba2-2.7B W8A8 model
        del graph, lm, states, ws, logits, tok
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        pl = run_prefill(args, dict(WORKLOADS["prefill27b"], name="prefill27b"), world, rank, local, emit=False)
        if pl is not None:
            prefill = {k: pl[k] for k in ("metric", "value", "unit", "ms_per_step", "config", "roofline",
                                          "roofline_gemm", "e2e", "gpu_launches", "cpu_baseline", "clocks")}
    if rank == 0:
        line = {"metric": "decode tok/s", "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "int8" if blk.a8 else "f32", "data": "synthetic",
                "config": {"workload": args.workload, "desc": wl["desc"], "model": wl.get("model", "Mamba2-8B-shaped"),
                           "global_batch": global_batch, "batch_per_gpu": B, "seq_len": 1, "layers": wl["layers"],
                           "vocab": wl["vocab"],
                           "parallelism": parallelism,
                           "l2": "inputs larger than L2 (weights+state stream every step), no flush",
                           "step_bytes": step_bytes,
                           "step_hbm_frac": step_bytes / (ms / 1e3) / 1e9 / hbm},
                "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": hbm,
                             "unit": "GB/s", "frac": achieved / hbm, "traffic": ncu_traffic(dom_name),
                             "peak_kind": pk_kind, "algorithmic_bytes_per_launch": dom_bytes,
                             "launch_ms": dom_ms},
                "cpu_baseline": res,
                "e2e": {"value": global_batch / (e2e_ms / 1e3), "unit": "tok/s", "h2d_bytes_per_step": B * 4,
                        "d2h_bytes_per_step": B * 4},
                "gpu_launches": launches_per_step * args.steps,
                "clocks": clk.summary(), "prefill": prefill}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="decode8b", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true", help="decode8b: skip the configs[1] prefill sub-record")
    ap.add_argument("--parallel", default="batch", choices=["batch", "heads"],
                    help="decode: batch-shard replicas (default) or head-shard tensor parallelism (NCCL all_reduce)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="decode: shard this many sequences over the ranks (strong scaling); default 64 per GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference_arm(args, wl, world, rank)
        return
    world, rank, local = dist_init()
    if "seq" in wl:   # prefill workloads
        run_prefill(args, wl, world, rank, local)
    else:
        run_decode(args, wl, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
