"""CPU: the C-ABI boundary (include/ssmquant_sm100.h) without touching a GPU.

* libssmquant_sm100.so builds for sm_100a, loads, and exports every entry point the
  header declares (and the ctypes table types exactly those);
* it carries sm_100a SASS (tcgen05 / TMA instructions present in the GEMM);
* the product path refuses CPU tensors (no CPU fallback) with the reference's
  exception classes.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ssmquant_sm100.h")


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2503_22879_b200 import _lib
    return _lib.load()


def header_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"\b(sq_[a-z0-9_]+)\s*\(", txt))


def test_header_declares_the_contract():
    syms = header_symbols()
    for s in ("sq_gemm_w8a8", "sq_gemm_w4a8", "sq_gemv_w4a16", "sq_conv1d_int8", "sq_conv1d_update_int8",
              "sq_ssd_scan_int8", "sq_selective_scan_int8", "sq_state_update_int8", "sq_gate_norm_had_quant",
              "sq_repack_w4", "sq_last_error", "sq_abi_version"):
        assert s in syms, s          # SURVEY §8(b) export list


def test_library_exports_every_declared_symbol(lib):
    from paper_2503_22879_b200 import _lib
    syms = header_symbols()
    assert syms == set(_lib.EXPORTS), syms ^ set(_lib.EXPORTS)
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(raw, s), s
    assert lib.sq_abi_version() == _lib.ABI_VERSION


def test_no_device_reports_unsupported(lib):
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert lib.sq_device_supported() == 0
    from paper_2503_22879_b200 import _lib
    msg = _lib.last_error()
    assert isinstance(msg, str)


def test_sass_is_sm100a_with_tcgen05_and_tma(lib):
    from paper_2503_22879_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTCIMMA" in sass or "UTCQMMA" in sass or "UTCHMMA" in sass, "tcgen05.mma missing"
    assert "UTMALDG" in sass or "UBLKCP" in sass, "TMA missing"
    assert "LDTM" in sass, "tcgen05.ld missing"


def test_ops_refuse_cpu_tensors(lib):
    from paper_2503_22879_b200 import errors, ops
    a = torch.zeros((4, 64), dtype=torch.int8)
    w = torch.zeros((8, 64), dtype=torch.int8)
    with pytest.raises(errors.LayoutError, match="no CPU fallback"):
        ops.gemm_w8a8(a, w, torch.ones(8), ops.EPI_F32)
    with pytest.raises(errors.LayoutError):
        ops.quantize_f32(torch.zeros((2, 8)), 0.1)
    assert issubclass(errors.LayoutError, errors.SsmQuantError)
    assert issubclass(errors.ShapeError, ValueError)


def test_status_mapping():
    from paper_2503_22879_b200 import errors
    assert isinstance(errors.status_error(-1, "x"), errors.ShapeError)
    assert isinstance(errors.status_error(-2, "x"), errors.LayoutError)
    assert isinstance(errors.status_error(-3, "x"), errors.KernelError)
    assert isinstance(errors.status_error(-4, "x"), RuntimeError)


def test_reference_package_alias():
    """`import ssmquant` resolves the reference module names to this implementation."""
    import ssmquant
    from ssmquant import errors, tensor
    assert tensor.__all__ == ["ShapeError", "as_f32", "require_finite", "matmul", "make_rng"]
    assert tensor.ShapeError is errors.ShapeError                 # D3 fixed
    with pytest.raises(errors.ArchiveError):                      # D4 fixed
        tensor.require_finite(np.array([np.inf], np.float32))
    assert np.array_equal(tensor.matmul([[1, 2], [3, 4]], [[5], [6]]), [[17], [39]])
    from oracle.tensor_core import make_rng as omr
    assert np.array_equal(tensor.make_rng(3, 1, 2).integers(0, 1 << 62, 8), omr(3, 1, 2).integers(0, 1 << 62, 8))
    assert ssmquant.__version__ == "0.1.0"
