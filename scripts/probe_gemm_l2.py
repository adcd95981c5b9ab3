"""Slice GEMM at the north-star shape (24 x 2048^3, bf16 out) vs cuBLAS, for the L2-bound question.

Usage: python scripts/probe_gemm_l2.py [stl|bmm|dense|all]  (ITERS env, default 30)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_12211_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
r, M, N, K = 24, 2048, 2048, 2048
n = int(os.environ.get("ITERS", "30"))


def timeit(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


what = sys.argv[1] if len(sys.argv) > 1 else "all"
out = {}
if what in ("stl", "all"):
    lib = _lib.load()
    a = torch.randn((r, M, K), device=dev).to(torch.bfloat16)
    b = torch.randn((r, N, K), device=dev).to(torch.bfloat16)
    c = torch.empty((r, M, N), device=dev, dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    ms = timeit(lambda: _lib.check(lib.stl_slice_gemm(a.data_ptr(), 0, b.data_ptr(), 0, c.data_ptr(),
                                                      1, 1, r, M, N, K, s)))
    ref = torch.bmm(a[:2].float(), b[:2].float().transpose(1, 2))
    err = ((c[:2].float() - ref).norm() / ref.norm()).item()
    out["stl"] = {"ms": ms, "tflops": 2 * r * M * N * K / ms / 1e9, "rel_err": err}
if what in ("bmm", "all"):
    a = torch.randn((r, M, K), device=dev).to(torch.bfloat16)
    b = torch.randn((r, K, N), device=dev).to(torch.bfloat16)
    ms = timeit(lambda: torch.bmm(a, b))
    out["cublas_bmm"] = {"ms": ms, "tflops": 2 * r * M * N * K / ms / 1e9}
if what in ("dense", "all"):
    a = torch.randn((8192, 8192), device=dev).to(torch.bfloat16)
    b = torch.randn((8192, 8192), device=dev).to(torch.bfloat16)
    ms = timeit(lambda: a @ b)
    out["cublas_dense8192"] = {"ms": ms, "tflops": 2 * 8192 ** 3 / ms / 1e9}
out["env"] = {k: v for k, v in os.environ.items() if k.startswith("STL_")}
print(json.dumps(out))
