"""Generate tests/golden/ fixtures by running the SHIPPED reference code.

Run in the dev container (needs /root/reference, read-only):
    python tests/golden/make_golden.py
The reference ships only `pkg/src/ssmquant/tensor.py` and `errors.py`;
its `matmul` (tensor.py:33-54) is the float-GEMM semantics every projection of the
SPEC block follows, so its outputs on seeded inputs are the golden vectors that pin
`oracle.tensor_core.matmul` and the exact integer GEMM `oracle.tensor_core.int_gemm`.
`make_rng` (tensor.py:57-69) is recorded as raising (defect D1); the fixed stream
the oracle uses instead (LEDGER G1) is recorded alongside, labelled as ours.
The fixtures are small and committed; nothing on the GPU box reads /root/reference.
"""
from __future__ import annotations

import importlib.util
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src/ssmquant"


def _load(name):
    spec = importlib.util.spec_from_file_location(f"ref_ssmquant_{name}", os.path.join(REF, f"{name}.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def main():
    t = _load("tensor")
    e = _load("errors")
    r = np.random.default_rng(20250329)
    cases = {}
    # SPEC.md:64-66 examples, run through the reference
    cases["spec_2x2_2x1"] = (np.array([[1, 2], [3, 4]], np.float32), np.array([[5], [6]], np.float32))
    cases["spec_1x0_0x1"] = (np.zeros((1, 0), np.float32), np.zeros((0, 1), np.float32))
    cases["spec_identity"] = (np.eye(2, dtype=np.float32), r.standard_normal((2, 2)).astype(np.float32))
    # float GEMMs at odd shapes
    cases["f32_5x7x3"] = (r.standard_normal((5, 7)).astype(np.float32), r.standard_normal((7, 3)).astype(np.float32))
    cases["f32_16x64x24"] = (r.standard_normal((16, 64)).astype(np.float32),
                             (r.standard_normal((64, 24)) * np.exp(r.uniform(-3, 3, (64, 1)))).astype(np.float32))
    # integer-valued operands (int8 activations x int8 / int4*sg weights): exact int32 accumulators
    cases["i8_8x512x12"] = (r.integers(-128, 128, (8, 512)).astype(np.float32),
                            r.integers(-127, 128, (512, 12)).astype(np.float32))
    cases["w4sg_4x256x6"] = (r.integers(-128, 128, (4, 256)).astype(np.float32),
                             (r.integers(-8, 8, (256, 6)) * r.integers(1, 16, (1, 6))).astype(np.float32))
    arrays = {}
    for k, (a, b) in cases.items():
        arrays[f"{k}.a"] = a
        arrays[f"{k}.b"] = b
        arrays[f"{k}.c"] = t.matmul(a, b)
    np.savez(os.path.join(HERE, "ref_matmul.npz"), **arrays)

    meta = {"source": "reference pkg/src/ssmquant/tensor.py executed by tests/golden/make_golden.py",
            "tensor_all": list(t.__all__)}
    try:
        t.make_rng(0)
        meta["make_rng_raises"] = None
    except Exception as ex:          # defect D1
        meta["make_rng_raises"] = f"{type(ex).__name__}: {ex}"
    try:
        t.require_finite(np.array([np.nan], np.float32))
        meta["require_finite_raises"] = None
    except Exception as ex:
        meta["require_finite_raises"] = type(ex).__name__
    try:
        t.matmul(np.zeros((2, 3), np.float32), np.zeros((2, 3), np.float32))
    except Exception as ex:
        meta["matmul_shape_error"] = type(ex).__name__
        meta["matmul_shape_error_is_valueerror"] = isinstance(ex, ValueError)
    meta["errors_hierarchy"] = {n: [b.__name__ for b in getattr(e, n).__mro__[1:]]
                                for n in ("SsmQuantError", "ShapeError", "LayoutError", "ArchiveError",
                                          "CalibrationError", "PipelineError")}
    # our fixed RNG stream (LEDGER G1), recorded so the oracle and the product stay in lock-step
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from oracle.tensor_core import make_rng
    meta["fixed_rng_first_u64"] = {f"{s}": [int(v) for v in make_rng(*s).integers(0, 2**63, 4)]
                                   for s in [(0,), (0, 1), (0, 1, 2), (0, 1, 2, 3), (7, 7, 7)]}
    with open(os.path.join(HERE, "ref_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
