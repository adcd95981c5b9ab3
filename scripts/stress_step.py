"""Stress: many config-2 forward+backward steps through the C ABI, one sync at the end (and
optionally per step with STRESS_SYNC=1), to catch intermittent kernel faults."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200.layer import LayerCache, backward_raw  # noqa: E402
from paper_2503_12211_b200.snf_operator import _forward  # noqa: E402

dev = torch.device("cuda")
T, R, M, K, N = 4, 24, 8192, 4096, 4096
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
w = torch.randn((R, N // T, K // T), device=dev).to(torch.bfloat16) * 0.03
x = torch.randn((M, K), device=dev).to(torch.bfloat16)
gy = torch.randn((M, N), device=dev).to(torch.bfloat16)
steps = int(os.environ.get("STRESS_STEPS", "500"))
sync_each = os.environ.get("STRESS_SYNC") == "1"
for i in range(steps):
    y, u, ye = _forward(x, w, snf, keep_cache=True)
    g = backward_raw(snf, w, LayerCache(x, u, ye), gy)
    if sync_each:
        torch.cuda.synchronize()
torch.cuda.synchronize()
print("stress ok", steps, float(g[0].abs().sum()))
