"""Micro-benchmark of the STL slice GEMM (stl_slice_gemm) at the bench shapes."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_12211_b200 import _lib

lib = _lib.load()
dev = torch.device("cuda")
shapes = {"cfg2_fwd": (24, 2048, 1024, 1024, 0, 0), "cfg2_gu": (24, 2048, 1024, 1024, 0, 1),
          "cfg2_gw": (24, 1024, 1024, 2048, 1, 1), "n8192": (24, 2048, 2048, 2048, 0, 0)}
sel = sys.argv[1:] or list(shapes)
for name in sel:
    r, M, N, K, al, bl = shapes[name]
    a = torch.randn((r, M, K) if al == 0 else (r, K, M), device=dev).to(torch.bfloat16)
    b = torch.randn((r, N, K) if bl == 0 else (r, K, N), device=dev).to(torch.bfloat16)
    c = torch.empty((r, M, N), device=dev, dtype=torch.float32)
    s = torch.cuda.current_stream().cuda_stream
    def run():
        _lib.check(lib.stl_slice_gemm(a.data_ptr(), al, b.data_ptr(), bl, c.data_ptr(), 0, 1, r, M, N, K, s))
    for _ in range(5): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = int(os.environ.get("ITERS", "20"))
    e0.record()
    for _ in range(n): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(json.dumps({"shape": name, "ms": ms, "tflops": 2 * r * M * N * K / ms / 1e9,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("STL_")}}))
