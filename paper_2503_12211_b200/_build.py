"""In-tree build of the STL CUDA library (libstl_b200.so) for sm_100a.

The library is a plain C-ABI shared object (include/stl_b200.h) built straight with nvcc —
no torch extension machinery — so it travels with the repo snapshot to the GPU box and is
loaded with ctypes by :mod:`paper_2503_12211_b200._lib`.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
LIB_NAME = "libstl_b200.so"
LIB_PATH = PKG / LIB_NAME

SOURCES = ["stl_capi.cu", "stl_slice_gemm.cu", "stl_transform.cu", "stl_transform4.cu",
           "stl_fused_gemm.cu", "stl_transform_mma.cu", "stl_stream.cu", "stl_tokens.cu"]
HEADERS = ["sm100_ptx.cuh", "sm100_pair_pipeline.cuh", "stl_internal.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    cand = [os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"]
    for c in cand:
        if c and Path(c).exists():
            return c
    raise RuntimeError("nvcc not found (set NVCC or install CUDA 12.9)")


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [REPO / "include" / "stl_b200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, obj: Path) -> subprocess.CompletedProcess:
    cmd = [nvcc(), *NVCC_FLAGS, *os.environ.get("STL_NVCC_EXTRA", "").split(), "-c", "-o",
           str(obj), str(src), "-I", str(REPO / "include")]
    return subprocess.run(cmd, capture_output=True, text=True)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every .cu (in parallel, one object each) and link one shared library (skips if
    up to date)."""
    if not force and not _stale():
        return LIB_PATH
    from concurrent.futures import ThreadPoolExecutor

    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    objs = [objdir / (Path(s).stem + ".o") for s in SOURCES]
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        procs = list(ex.map(lambda so: _compile(CSRC / so[0], so[1]), zip(SOURCES, objs)))
    log = PKG / "build.log"
    text = "".join(" ".join(p.args) + "\n" + p.stdout + p.stderr for p in procs)
    bad = [p for p in procs if p.returncode != 0]
    if not bad:
        link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                str(LIB_PATH), *map(str, objs), "-lcudart_static"]
        lp = subprocess.run(link, capture_output=True, text=True)
        text += " ".join(link) + "\n" + lp.stdout + lp.stderr
        if lp.returncode != 0:
            bad = [lp]
    log.write_text(text)
    if bad:
        raise RuntimeError(f"nvcc failed ({bad[0].returncode}); see {log}\n{bad[0].stderr[-4000:]}")
    if verbose:
        print(text)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force=True, verbose=True))
