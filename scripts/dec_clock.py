"""Decode (8192^3) SM clock and loop time right after the slice GEMM vs after idle (probe
library, STL_STREAM_DEBUG=1: the kernel records clock64 / globaltimer over its unit loop)."""
import os
import sys
import time

os.environ.setdefault("STL_STREAM_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_12211_b200 import _lib  # noqa: E402
os.environ.setdefault("STL_LIB", str(_lib.PROBE_LIB_PATH))
import torch  # noqa: E402
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
s = torch.cuda.current_stream().cuda_stream
gemm = lambda: _lib.check(lib.stl_slice_gemm(u.data_ptr(), 0, w.data_ptr(), 0, ye.data_ptr(), 1, 1, R, b, b, b, s))
dec = lambda: _lib.check(lib.stl_decode(ye.data_ptr(), 1, b, b, R, snf.d.data_ptr(), T, y.data_ptr(), 1, n, s))
for tag, pred in (("idle", None), ("gemm", gemm), ("idle", None), ("gemm", gemm), ("gemm", gemm)):
    time.sleep(0.1)
    if pred:
        pred()
    print(tag, flush=True)
    dec()
    torch.cuda.synchronize()
