import os, sys
sys.path.insert(0, "/root/repo")
os.chdir(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2503_22879_b200 import ops
def timeit(fn, reps=20):
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for i in range(reps): fn(i)
    torch.cuda.current_stream().wait_stream(s); g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000
for name, M, N, K in (("in_proj", 64, 18560, 4096), ("out_proj", 64, 4096, 8192)):
    a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device="cuda")
    out = torch.empty((M, N), dtype=torch.float32, device="cuda")
    for nbuf in (1, 8):
        w4 = [torch.randint(0, 256, (ops.w4_bytes(N, K),), dtype=torch.uint8, device="cuda") for _ in range(nbuf)]
        ws = [ops.tile_group_scales(torch.rand(N, K // 128, device="cuda") * 1e-2 + 1e-3) for _ in range(nbuf)]
        t = timeit(lambda i: ops.gemm_w4a8(a, w4[i % nbuf], ws[i % nbuf], 128, 0.01, N, ops.EPI_F32, out))
        print(f"{name} nbuf={nbuf} ({'L2-resident' if nbuf == 1 else 'HBM'}): {t:.1f} us", flush=True)
