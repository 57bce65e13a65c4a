"""Time gate_norm_had_quant at the 2.7B prefill shape (16384 x 5120) for probe builds
(probe/probe_<name>.so); codes compared with the first variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import _lib, ops  # noqa: E402

M, D = 16384, 5120
g = torch.Generator(device="cuda")
g.manual_seed(1)
y = torch.randn((M, D), device="cuda", generator=g)
gam = torch.rand(D, device="cuda", generator=g) + 0.5
ref = None
for name in sys.argv[1:]:
    _lib._lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", f"probe_{name}.so"))
    out = torch.empty((M, D), dtype=torch.int8, device="cuda")
    for _ in range(3):
        ops.gate_norm_had_quant(y, gam, 1e-5, 0.05, True, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ops.gate_norm_had_quant(y, gam, 1e-5, 0.05, True, out)
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    d = (out.int() - ref.int()).abs()
    print(f"{name:8s} {e0.elapsed_time(e1) * 100:.1f} us  codes max|d| {d.max().item()} "
          f"frac {(d > 0).float().mean().item():.2e}", flush=True)
