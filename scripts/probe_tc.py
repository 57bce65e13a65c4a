"""Time the W8A8 tcgen05 GEMM probe variants (probe/probe_<name>.so) on the prefill projection
shapes: Mamba1 2.8B at B*T = 1024 (configs[4]) and Mamba2 2.7B at 16384 tokens.  Distinct weight
buffers per launch (weights stream from HBM), launches replayed from a CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import _lib, ops  # noqa: E402

SHAPES = [("m1 in_proj", 1024, 10240, 2560, ops.EPI_QUANT), ("m1 x_proj", 1024, 192, 5120, ops.EPI_QUANT),
          ("m1 dt_proj", 1024, 5120, 160, ops.EPI_QUANT), ("m1 out_proj", 1024, 2560, 5120, ops.EPI_RESID),
          ("m2 in_proj 4k", 4096, 10576, 2560, ops.EPI_QUANT), ("m2 in_proj 16k", 16384, 10576, 2560, ops.EPI_QUANT),
          ("m2 out_proj 16k", 16384, 2560, 5120, ops.EPI_RESID)]


def timeit(fn, reps=10):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                fn(i)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dev = "cuda"
only = os.environ.get("ONLY")
data = []
for name, M, N, K, epi in SHAPES:
    if only and only not in name:
        continue
    a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev)
    alpha = torch.rand(N, device=dev) * 1e-3
    cs = torch.rand(N, device=dev) + 0.5
    nbuf = max(1, min(8, int(1e9 // (N * K))))
    w8 = [torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev) for _ in range(nbuf)]
    out = torch.zeros((M, N), dtype=torch.float32 if epi == ops.EPI_RESID else torch.int8, device=dev)
    data.append((name, M, N, K, epi, a, alpha, cs, w8, nbuf, out))
ref = {}
for v in sys.argv[1:]:
    _lib._lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", f"probe_{v}.so"))
    for name, M, N, K, epi, a, alpha, cs, w8, nbuf, out in data:
        def run(i):
            ops.gemm_w8a8(a, w8[i % nbuf], alpha, epi, out, cs if epi == ops.EPI_QUANT else None)
        if epi == ops.EPI_RESID:
            out.zero_()
            run(0)
            chk = out.clone()
        else:
            run(0)
            chk = out.float()
        bad = ""
        if name in ref and not torch.equal(chk, ref[name]):
            bad = f"  MISMATCH max {(chk - ref[name]).abs().max().item():.3g}"
        ref.setdefault(name, chk)
        t = timeit(run)
        print(f"{v:8s} {name:16s} {t*1e3:8.1f} us {2.0*M*N*K/t/1e9:7.1f} TOPS{bad}", flush=True)
