import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2503_22879_b200 import ops
from paper_2503_22879_b200.ssm_block import pack_u4_host
M, N, K, reps = (int(v) for v in sys.argv[1:5])
r = np.random.default_rng(0)
modes = [int(v) for v in sys.argv[5].split(',')] if len(sys.argv) > 5 else [1, 2]
for mode in modes:
    ops.set_gemm_mode(mode)
    bad = 0
    for it in range(reps):
        a = r.integers(-128, 128, (M, K)).astype(np.int8)
        codes = r.integers(-8, 8, (N, K)).astype(np.int8)
        sg = r.integers(1, 16, (N, K // 128)).astype(np.int8)
        tw = ops.repack_w4(torch.as_tensor(pack_u4_host(codes), device="cuda"), N, K)
        w8 = (codes.astype(np.int64).reshape(N, K // 128, 128) * sg[:, :, None]).reshape(N, K)
        acc = a.astype(np.int64) @ w8.T
        got = ops.gemm_w4a8(torch.as_tensor(a, device="cuda"), tw, torch.as_tensor(sg, device="cuda"), 128,
                            torch.ones(N, device="cuda"), N, ops.EPI_I32).cpu().numpy()
        if not np.array_equal(got, acc):
            bad += 1
            d = np.argwhere(got != acc)
            print(f"  mode {mode} it {it}: {len(d)} mismatches; first {d[:3].tolist()} rows/cols distinct "
                  f"{len(set(d[:,0]))}/{len(set(d[:,1]))}", flush=True)
    print("mode", mode, "bad", bad, "of", reps, flush=True)
