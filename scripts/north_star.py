"""The north-star comparison alone: 8192^3 bf16 STL forward (t=4, r=24) vs cuBLAS, burst
(short alternating blocks after idle) and sustained (long alternating blocks), as bench.py."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda")
T, R, n = 4, 24, 8192
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
wf = stl.weights_to_planes(stl.encode_tiles(torch.randn((n, n), device=dev) / n ** 0.5, snf.e_w, T),
                           dtype=torch.bfloat16)
xf = torch.randn((n, n), device=dev).to(torch.bfloat16)
uf = torch.empty((R, n // T, n // T), dtype=torch.bfloat16, device=dev)
sf = torch.empty((int(lib.stl_forward_scratch_bytes(n, n, n, T, R, _lib.STL_BF16)),), dtype=torch.uint8,
                 device=dev)
yf = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
wdf = torch.randn((n, n), device=dev).to(torch.bfloat16)
ydf = torch.empty((n, n), device=dev, dtype=torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream


def fwd():
    _lib.check(lib.stl_forward(xf.data_ptr(), n, n, n, wf.data_ptr(), n, snf.e_x.data_ptr(),
                               snf.d.data_ptr(), T, R, _lib.STL_BF16, yf.data_ptr(), n,
                               uf.data_ptr(), None, sf.data_ptr(), sf.numel(), s))


def cub():
    torch.matmul(xf, wdf, out=ydf)


def timed(fn, k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


for _ in range(5):
    fwd(); cub()
sb, cb = [], []
for _ in range(7):
    time.sleep(0.06)
    sb.append(timed(fwd, 10))
    time.sleep(0.06)
    cb.append(timed(cub, 10))
ss, cs = [], []
for _ in range(5):
    ss.append(timed(fwd, 100))
    cs.append(timed(cub, 100))
med = statistics.median
print(json.dumps({"burst": {"stl_ms": med(sb), "cublas_ms": med(cb), "speedup": med(cb) / med(sb),
                            "stl": [round(v, 4) for v in sb], "cublas": [round(v, 4) for v in cb]},
                  "sustained": {"stl_ms": med(ss), "cublas_ms": med(cs), "speedup": med(cs) / med(ss),
                                "stl": [round(v, 4) for v in ss], "cublas": [round(v, 4) for v in cs]},
                  "lib": os.environ.get("STL_LIB", "product")}), flush=True)
