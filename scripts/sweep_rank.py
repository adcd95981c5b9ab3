"""BASELINE configs[2]: rank / tile sweep of the STL forward at M = K = N = 8192, bf16.

    python scripts/sweep_rank.py > profiles/r01_rank_sweep.jsonl

t in {2, 4}, r in {16, 24, 32} (random N(0, 0.25) triples) plus r = 49 at t = 4 (Strassen x
Strassen, exact). For every point: the forward (encode -> slice GEMMs -> decode) time, the
slice GEMM's TF/s and fraction of the measured sustained bf16 peak, the dense-equivalent
TF/s and the ratio to cuBLAS' dense 8192^3 GEMM timed the same way.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200 import _lib  # noqa: E402
from paper_2503_12211_b200.snf_operator import _forward  # noqa: E402


def timed(fn, n):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    n = 8192
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("bf16_tflops_sustained", 1400.0)
    lib = _lib.load()
    dev = torch.device("cuda")
    x = torch.randn(n, n, device=dev).to(torch.bfloat16)
    wd = torch.randn(n, n, device=dev).to(torch.bfloat16)
    yd = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
    cub = timed(lambda: torch.matmul(x, wd, out=yd), 10)
    points = [(2, 16), (2, 24), (2, 32), (4, 16), (4, 24), (4, 32), (4, 49)]
    for t, r in points:
        if r == 49:
            snf = stl.strassen_rank49().to(dev)
        else:
            snf = stl.random_gaussian_init(t, r, np.random.Generator(np.random.PCG64(r)), scale=0.5).to(dev)
        w_planes = stl.weights_to_planes(stl.encode_tiles(wd.float() / n ** 0.5, snf.e_w, t),
                                         dtype=torch.bfloat16)
        ms = timed(lambda: _forward(x, w_planes, snf), 5)
        lib.stl_profile_reset()
        lib.stl_profile_enable(1)
        _forward(x, w_planes, snf)
        torch.cuda.synchronize()
        lib.stl_profile_enable(0)
        recs = _lib.profile_records()
        gemm_ms = sum(m for name, m, _ in recs if name.startswith("slice_gemm"))
        gemm_flops = 2.0 * r * (n // t) ** 3
        del w_planes
        torch.cuda.empty_cache()
        print(json.dumps({
            "t": t, "r": r, "init": "strassen49" if r == 49 else "gaussian",
            "stl_fwd_ms": ms, "cublas_dense_ms": cub, "speedup_vs_cublas": cub / ms,
            "dense_equiv_tflops": 2.0 * n ** 3 / (ms * 1e-3) / 1e12,
            "gemm_ms": gemm_ms, "gemm_tflops": gemm_flops / (gemm_ms * 1e-3) / 1e12,
            "gemm_frac_of_sustained_peak": gemm_flops / (gemm_ms * 1e-3) / 1e12 / peak,
            "flops_ratio_dense_over_stl": 2.0 * n ** 3 / gemm_flops,
            "kernels_ms": {name: round(m, 4) for name, m, _ in recs}}), flush=True)


if __name__ == "__main__":
    main()
