"""Drop-in alias of the reference package name `ssmquant` (pkg/pyproject.toml:6).

`import ssmquant.quantizer` etc. resolve to the B200 implementation in
`paper_2503_22879_b200`; see INTEGRATION.md.
"""
import importlib
import sys

_MODULES = ("errors", "tensor", "quantizer", "hadamard", "ssm_block", "calibrate", "reorder", "archive", "cli",
            "model", "ops")

for _m in _MODULES:
    try:
        globals()[_m] = sys.modules[f"{__name__}.{_m}"] = importlib.import_module(f"paper_2503_22879_b200.{_m}")
    except ModuleNotFoundError as e:          # module not written yet
        if e.name != f"paper_2503_22879_b200.{_m}":
            raise

from paper_2503_22879_b200 import errors, tensor  # noqa: E402,F401

__version__ = "0.1.0"
