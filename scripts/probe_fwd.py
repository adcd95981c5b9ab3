"""North-star forward timing: STL forward at 8192^3 t=4 r=24 bf16 vs cuBLAS dense (ITERS, SEEDS)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200.snf_operator import _forward  # noqa: E402

dev = torch.device("cuda")
T, R = 4, int(os.environ.get("RANK_R", "24"))
M = K = N = int(os.environ.get("SIZE", "8192"))
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
x = torch.randn((M, K), device=dev).to(torch.bfloat16)
w = (torch.randn((R, N // T, K // T), device=dev) * 0.05).to(torch.bfloat16)
a = torch.randn((M, K), device=dev).to(torch.bfloat16)
b = torch.randn((K, N), device=dev).to(torch.bfloat16)
n = int(os.environ.get("ITERS", "20"))


def timeit(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(x.elapsed_time(y) for x, y in ts)
    return v[len(v) // 2], v[0]


stl_med, stl_min = timeit(lambda: _forward(x, w, snf))
cub_med, cub_min = timeit(lambda: a @ b)
y = _forward(x, w, snf)
ref = stl.stl_batched(x[:256].float(), w.float().permute(2, 1, 0), snf)
err = ((y[:256].float() - ref).norm() / ref.norm()).item()
print(json.dumps({"stl_ms": stl_med, "stl_min": stl_min, "cublas_ms": cub_med, "cublas_min": cub_min,
                  "speedup": cub_med / stl_med, "rel_err_vs_fp32_rows": err,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("STL_")}}))
