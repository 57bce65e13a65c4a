import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2503_22879_b200 import ops
mode, M, N, K = (int(v) for v in sys.argv[1:5])
ops.set_gemm_mode(mode)
r = np.random.default_rng(0)
a = r.integers(-128, 128, (M, K)).astype(np.int8)
codes = r.integers(-8, 8, (N, K)).astype(np.int8)
sg = r.integers(1, 16, (N, K // 128)).astype(np.int8)
from paper_2503_22879_b200.ssm_block import pack_u4_host
tw = ops.repack_w4(torch.as_tensor(pack_u4_host(codes), device="cuda"), N, K)
ok = np.array_equal(ops.unpack_w4(tw, N, K).cpu().numpy(), pack_u4_host(codes))
w8 = (codes.astype(np.int64).reshape(N, K // 128, 128) * sg[:, :, None]).reshape(N, K)
acc = a.astype(np.int64) @ w8.T
got = ops.gemm_w4a8(torch.as_tensor(a, device="cuda"), tw, torch.as_tensor(sg, device="cuda"), 128,
                    torch.ones(N, device="cuda"), N, ops.EPI_I32).cpu().numpy()
print("mode", mode, M, N, K, "roundtrip", ok, "exact", np.array_equal(got, acc), "maxdiff", np.abs(got - acc).max(), flush=True)
