"""Slice-GEMM result check at bench shapes against torch.bmm (fp32 accumulate of bf16 inputs)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_12211_b200 import _lib

lib = _lib.load()
dev = torch.device("cuda")
shapes = {"cfg2_fwd": (24, 2048, 1024, 1024), "n8192": (24, 2048, 2048, 2048),
          "odd": (5, 1000, 520, 264)}
for name, (r, M, N, K) in shapes.items():
    g = torch.Generator(device=dev).manual_seed(0)
    a = torch.randn((r, M, K), device=dev, generator=g).to(torch.bfloat16)
    b = torch.randn((r, N, K), device=dev, generator=g).to(torch.bfloat16)
    c = torch.full((r, M, N), float("nan"), device=dev, dtype=torch.float32)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.stl_slice_gemm(a.data_ptr(), 0, b.data_ptr(), 0, c.data_ptr(), 0, 1, r, M, N, K, s))
    ref = torch.bmm(a.float(), b.float().transpose(1, 2))
    err = float((c - ref).norm() / ref.norm())
    print(json.dumps({"shape": name, "rel_err": err, "nan": bool(torch.isnan(c).any()),
                      "env": {k: v for k, v in os.environ.items() if k.startswith("STL_")}}))
