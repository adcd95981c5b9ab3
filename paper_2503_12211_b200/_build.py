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
# The probe build: the same sources with -DSTL_PROBES, whose STL_* environment switches
# (scripts/) select A/B variants and timers. The product library never reads the environment.
PROBE_LIB_PATH = PKG / "libstl_b200_probe.so"

SOURCES = ["stl_capi.cu", "stl_slice_gemm.cu", "stl_transform.cu", "stl_transform2.cu",
           "stl_transform4.cu",
           "stl_transform_mma.cu", "stl_stream.cu", "stl_stream_tc.cu", "stl_tokens.cu"]
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


def _stale(lib: Path) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [REPO / "include" / "stl_b200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, obj: Path, extra: list[str]) -> subprocess.CompletedProcess:
    cmd = [nvcc(), *NVCC_FLAGS, *extra, *os.environ.get("STL_NVCC_EXTRA", "").split(), "-c",
           "-o", str(obj), str(src), "-I", str(REPO / "include")]
    return subprocess.run(cmd, capture_output=True, text=True)


def build(force: bool = False, verbose: bool = False, probes: bool = True) -> Path:
    """Compile every .cu (in parallel, one object each) and link libstl_b200.so — and, with
    `probes`, libstl_b200_probe.so (-DSTL_PROBES) — skipping libraries that are up to date."""
    from concurrent.futures import ThreadPoolExecutor

    variants = [(LIB_PATH, PKG / "build", [])]
    if probes:
        variants.append((PROBE_LIB_PATH, PKG / "build" / "probe", ["-DSTL_PROBES"]))
    todo = [v for v in variants if force or _stale(v[0])]
    if not todo:
        return LIB_PATH
    jobs = []
    for lib, objdir, extra in todo:
        objdir.mkdir(parents=True, exist_ok=True)
        for src in SOURCES:
            jobs.append((CSRC / src, objdir / (Path(src).stem + ".o"), extra))
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 8)) as ex:
        procs = list(ex.map(lambda j: _compile(*j), jobs))
    log = PKG / "build.log"
    text = "".join(" ".join(p.args) + "\n" + p.stdout + p.stderr for p in procs)
    bad = [p for p in procs if p.returncode != 0]
    if not bad:
        for lib, objdir, _ in todo:
            objs = [str(objdir / (Path(src).stem + ".o")) for src in SOURCES]
            link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                    str(lib), *objs, "-lcudart_static"]
            lp = subprocess.run(link, capture_output=True, text=True)
            text += " ".join(link) + "\n" + lp.stdout + lp.stderr
            if lp.returncode != 0:
                bad = [lp]
                break
    log.write_text(text)
    if bad:
        raise RuntimeError(f"nvcc failed ({bad[0].returncode}); see {log}\n{bad[0].stderr[-4000:]}")
    if verbose:
        print(text)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force=True, verbose=True))
