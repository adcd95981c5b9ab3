"""C-ABI checks that need no GPU: the library loads, exports exactly the symbols
include/stl_b200.h declares, and rejects bad arguments with the reference's error classes
before touching the device."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2503_12211_b200 import _lib
from paper_2503_12211_b200.dense_core import ShapeError

HEADER = Path(__file__).resolve().parent.parent / "include" / "stl_b200.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"STL_API\s+[\w\s\*]+?\b(stl_\w+)\s*\(", text)))


def test_header_declares_all_bound_symbols():
    assert header_symbols() == sorted(_lib.SIGNATURES)


def test_library_exports_every_header_symbol(lib_path):
    lib = ctypes.CDLL(str(lib_path))
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_version_and_limits():
    lib = _lib.load()
    assert lib.stl_version().decode().startswith("stl_b200")
    assert lib.stl_max_rank() >= 49
    assert lib.stl_reduce_workspace_floats(24, 4) >= 24 * 16


def test_status_mapping_without_gpu():
    lib = _lib.load()
    # tile size 3 is not a supported kernel instantiation -> NotImplementedError
    st = lib.stl_encode(None, 0, 12, 12, 12, None, 3, 4, None, 0, None)
    with pytest.raises(NotImplementedError):
        _lib.check(st)
    # t does not divide the shape -> ShapeError (dense_core.py:70-74 semantics)
    st = lib.stl_encode(None, 0, 10, 8, 8, None, 4, 4, None, 0, None)
    with pytest.raises(ShapeError, match="does not divide"):
        _lib.check(st)
    # r = 0 -> ShapeError like SnfTriple.__post_init__ (snf_operator.py:60-61)
    st = lib.stl_forward(None, 8, 8, 8, None, 8, None, None, 4, 0, 0, None, 8, None, None, None, 0,
                         None)
    with pytest.raises(ShapeError):
        _lib.check(st)
    # batch not divisible by t -> ShapeError (toy_network.py:78-79)
    st = lib.stl_forward(None, 6, 8, 8, None, 8, None, None, 4, 4, 0, None, 8, None, None, None, 0,
                         None)
    with pytest.raises(ShapeError, match="batch"):
        _lib.check(st)
    # bad dtype -> ValueError
    st = lib.stl_slice_gemm(None, 0, None, 0, None, 7, 0, 1, 8, 8, 8, None)
    with pytest.raises(ValueError):
        _lib.check(st)
    # zero-sized problems are no-ops
    assert lib.stl_slice_gemm(None, 0, None, 0, None, 0, 0, 4, 0, 8, 8, None) == 0


def test_fused_step_ex_formats_without_gpu():
    """stl_fused_step_ex: bf16 encoded activations require bf16 weights (ValueError before any
    launch); invalid dtypes are ValueErrors too."""
    lib = _lib.load()
    st = lib.stl_fused_step_ex(None, _lib.STL_BF16, 4, 64, None, 4, None, None, 4, 24,
                               _lib.STL_F32, None, _lib.STL_F32, None, None, None)
    with pytest.raises(ValueError, match="bf16"):
        _lib.check(st)
    st = lib.stl_fused_step_ex(None, 9, 4, 64, None, 4, None, None, 4, 24, _lib.STL_BF16, None,
                               _lib.STL_BF16, None, None, None)
    with pytest.raises(ValueError):
        _lib.check(st)
