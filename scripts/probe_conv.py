"""Time the int8 prefill conv (sq_conv1d_int8) at the 2.7B prefill shape (8 x 2048 tokens,
5376 channels) for probe builds (probe/probe_<name>.so); codes and cache compared with the first."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import _lib, ops  # noqa: E402

B, T, C, K = 8, 2048, 5376, 4
g = torch.Generator(device="cuda")
g.manual_seed(2)
x = torch.randint(-128, 128, (B * T, C), dtype=torch.int8, device="cuda", generator=g)
w = torch.randn((C, K), device="cuda", generator=g) * 0.3
b = torch.randn(C, device="cuda", generator=g) * 0.05
s_in = torch.rand(C, device="cuda", generator=g) * 0.04 + 0.01
s_out = torch.rand(C, device="cuda", generator=g) * 0.04 + 0.01
cache0 = torch.randint(-128, 128, (B, K - 1, C), dtype=torch.int8, device="cuda", generator=g)
# saturating inputs too: a few channels with a tiny output scale
s_out[:64] = 1e-4
ref = None
for name in sys.argv[1:]:
    _lib._lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", f"probe_{name}.so"))
    out = torch.empty((B * T, C), dtype=torch.int8, device="cuda")
    for _ in range(3):
        ops.conv1d_int8(x, w, b, s_in, s_out, B, T, cache0.clone(), True, out)
    torch.cuda.synchronize()
    caches = [cache0.clone() for _ in range(10)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(10):
        ops.conv1d_int8(x, w, b, s_in, s_out, B, T, caches[i], True, out)
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = (out.clone(), caches[0].clone())
    print(f"{name:8s} {e0.elapsed_time(e1) * 100:.1f} us  codes equal {torch.equal(out, ref[0])} "
          f"cache equal {torch.equal(caches[0], ref[1])}", flush=True)
