"""The 8192^3 bf16 STL forward (north-star shape) run a few times, for profilers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200.snf_operator import _forward  # noqa: E402

dev = torch.device("cuda")
T, R, n = 4, 24, 8192
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
x = torch.randn((n, n), device=dev).to(torch.bfloat16)
w = torch.randn((R, n // T, n // T), device=dev).to(torch.bfloat16)
for _ in range(int(os.environ.get("ITERS", "4"))):
    _forward(x, w, snf)
torch.cuda.synchronize()
