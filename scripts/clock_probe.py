"""Effective SM clock right after different kernels: times torch.cuda._sleep(N cycles) (a
clock64 spin) launched behind them. One JSON line: MHz = N / duration."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_12211_b200 import _lib  # noqa: E402
import paper_2503_12211_b200 as stl  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda")
T, R, n = 4, 24, 8192
b = n // T
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
x = torch.randn((n, n), device=dev).to(torch.bfloat16)
u = torch.empty((R, b, b), dtype=torch.bfloat16, device=dev)
w = (torch.randn((R, b, b), device=dev) * 0.02).to(torch.bfloat16)
ye = torch.empty((R, b, b), dtype=torch.bfloat16, device=dev)
y = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
wd = torch.randn((n, n), device=dev).to(torch.bfloat16)
yd = torch.empty((n, n), device=dev, dtype=torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream
enc = lambda: _lib.check(lib.stl_encode(x.data_ptr(), 1, n, n, n, snf.e_x.data_ptr(), T, R, u.data_ptr(), 1, s))
gemm = lambda: _lib.check(lib.stl_slice_gemm(u.data_ptr(), 0, w.data_ptr(), 0, ye.data_ptr(), 1, 1, R, b, b, b, s))
dec = lambda: _lib.check(lib.stl_decode(ye.data_ptr(), 1, b, b, R, snf.d.data_ptr(), T, y.data_ptr(), 1, n, s))
cub = lambda: torch.matmul(x, wd, out=yd)
N = 40000  # ~20 us at 1965 MHz
out = {}
for name, pred in (("idle", None), ("gemm", gemm), ("cublas", cub), ("dec", dec), ("enc", enc),
                   ("gemm_x3", lambda: (gemm(), gemm(), gemm()))):
    mhz = []
    for _ in range(10):
        time.sleep(0.05)
        if pred:
            pred()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.cuda._sleep(N)
        e1.record()
        e2 = torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(N)
        e2.record()
        torch.cuda.synchronize()
        mhz.append((N / (e0.elapsed_time(e1) * 1e3), N / (e1.elapsed_time(e2) * 1e3)))
    mhz.sort()
    out[name] = [round(mhz[5][0]), round(mhz[5][1])]
print(json.dumps({"sm_mhz_first_and_second_20us_after": out}), flush=True)
