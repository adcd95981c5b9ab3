"""ctypes binding of the C ABI in ``include/stl_b200.h`` (libstl_b200.so).

This is the reference-side binding a maintainer of the (pure-Python) reference would add:
plain pointers, sizes and a stream handle cross the boundary, no torch types. There is no
CPU fallback: if the shared library or a CUDA device is missing, every operator raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_int, c_int64, c_void_p, c_char_p
from pathlib import Path

from .dense_core import ShapeError

LIB_PATH = Path(__file__).resolve().with_name("libstl_b200.so")
# the probe build (-DSTL_PROBES: STL_* environment A/B switches), for scripts/ and one stress test
PROBE_LIB_PATH = LIB_PATH.with_name("libstl_b200_probe.so")

STL_F32 = 0
STL_BF16 = 1
STL_F24 = 2  # intermediate format of the bf16 path's fp32 slice products (see stl_cache_bytes)
STL_PROD_AUTO = -1  # slice-product format chosen per shape (include/stl_b200.h)
STL_K_MAJOR = 0
STL_MN_MAJOR = 1

# Every exported symbol of include/stl_b200.h with its ctypes signature.
SIGNATURES = {
    "stl_version": ([], c_char_p),
    "stl_last_error": ([], c_char_p),
    "stl_max_rank": ([], c_int),
    "stl_reduce_workspace_floats": ([c_int, c_int], c_int64),
    "stl_encode": ([c_void_p, c_int, c_int64, c_int64, c_int64, c_void_p, c_int, c_int,
                    c_void_p, c_int, c_void_p], c_int),
    "stl_decode": ([c_void_p, c_int, c_int64, c_int64, c_int, c_void_p, c_int, c_void_p, c_int,
                    c_int64, c_void_p], c_int),
    "stl_slice_gemm": ([c_void_p, c_int, c_void_p, c_int, c_void_p, c_int, c_int, c_int,
                        c_int64, c_int64, c_int64, c_void_p], c_int),
    "stl_forward_scratch_bytes": ([c_int64, c_int64, c_int64, c_int, c_int, c_int], c_int64),
    "stl_cache_bytes": ([c_int64, c_int64, c_int64, c_int, c_int, c_int], c_int64),
    "stl_cache_bytes_ex": ([c_int64, c_int64, c_int64, c_int, c_int, c_int, c_int], c_int64),
    "stl_cache_format": ([c_int64, c_int64, c_int64, c_int, c_int, c_int, c_int], c_int),
    "stl_forward_ex": ([c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                        c_void_p, c_int, c_int, c_int, c_void_p, c_int64, c_void_p, c_void_p,
                        c_void_p, c_int64, c_int, c_void_p], c_int),
    "stl_backward_ex": ([c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                         c_void_p, c_void_p, c_int, c_int64, c_int64, c_int64, c_int, c_int,
                         c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                         c_void_p, c_void_p, c_int, c_void_p, c_void_p], c_int),
    "stl_forward": ([c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                     c_int, c_int, c_int, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                     c_int64, c_void_p], c_int),
    
    "stl_backward": ([c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                      c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_int, c_int,
                      c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                      c_void_p, c_void_p], c_int),
    "stl_fused_step": ([c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int,
                        c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p], c_int),
    "stl_fused_step_ex": ([c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                           c_void_p, c_int, c_int, c_int, c_void_p, c_int, c_void_p, c_void_p,
                           c_void_p], c_int),
    "stl_token_pad": ([c_void_p, c_int, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64,
                       c_void_p], c_int),
    "stl_token_unpad": ([c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int, c_int64, c_int64,
                         c_void_p], c_int),
    "stl_token_fold": ([c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p,
                        c_int64, c_void_p], c_int),
    "stl_token_fold_ws_floats": ([c_int64, c_int64, c_int64, c_int], c_int64),
    "stl_token_fold_backward": ([c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p,
                                 c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_void_p], c_int),
    "stl_profile_enable": ([c_int], c_int),
    "stl_profile_reset": ([], c_int),
    "stl_profile_count": ([], c_int),
    "stl_profile_get": ([c_int, ctypes.POINTER(c_char_p), ctypes.POINTER(ctypes.c_float),
                         ctypes.POINTER(c_int)], c_int),
}

_lib = None


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # STL_LIB: load another build of the library (A/B measurements)
    p = Path(path) if path is not None else Path(os.environ.get("STL_LIB") or LIB_PATH)
    if not p.exists():
        raise ImportError(
            f"STL CUDA library not found at {p}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = lib
    return lib


class StlCudaError(RuntimeError):
    """A CUDA launch inside the STL library failed."""


def check(status: int) -> None:
    """Map a C status code to the reference's exception classes."""
    if status == 0:
        return
    msg = (load().stl_last_error() or b"").decode(errors="replace")
    if status == 1:
        raise ShapeError(msg)
    if status == 2:
        raise ValueError(msg)
    if status == 3:
        raise IndexError(msg)
    if status == 5:
        raise NotImplementedError(msg)
    raise StlCudaError(msg)


def profile_records() -> list[tuple[str, float, int]]:
    """(name, ms, launches) of every record since the last stl_profile_reset (sync first)."""
    lib = load()
    out = []
    name = c_char_p()
    ms = ctypes.c_float()
    n = c_int()
    for i in range(lib.stl_profile_count()):
        check(lib.stl_profile_get(i, ctypes.byref(name), ctypes.byref(ms), ctypes.byref(n)))
        out.append((name.value.decode(), float(ms.value), int(n.value)))
    return out
