"""One 8192^3 (t=4, r=24) bf16 encode and decode through the C ABI, a few times (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda")
T, R, n = 4, 24, 8192
b = n // T
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
xf = torch.randn((n, n), device=dev).to(torch.bfloat16)
uf = torch.empty((R, b, b), dtype=torch.bfloat16, device=dev)
ye = torch.randn((R, b, b), device=dev).to(torch.bfloat16)
y2 = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.check(lib.stl_encode(xf.data_ptr(), 1, n, n, n, snf.e_x.data_ptr(), T, R, uf.data_ptr(), 1, s))
    _lib.check(lib.stl_decode(ye.data_ptr(), 1, b, b, R, snf.d.data_ptr(), T, y2.data_ptr(), 1, n, s))
torch.cuda.synchronize()
