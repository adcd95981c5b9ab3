"""Cache-less forward accuracy and time: bf16 slice products (default) vs F24 / fp32 products
(forced with stl_forward_ex) at BASELINE shapes; error vs a float64 restatement on the same bf16
inputs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200 import _lib  # noqa: E402
from paper_2503_12211_b200.snf_operator import _forward  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda")
T = 4
for (M, K, N, R) in ((8192, 8192, 8192, 24), (8192, 4096, 4096, 24), (4096, 4096, 4096, 49)):
    snf = (stl.strassen_rank49() if R == 49 else
           stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5)).to(dev)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
    w0 = torch.randn((K, N), device=dev, generator=g) / K ** 0.5
    w = stl.weights_to_planes(stl.encode_tiles(w0, snf.e_w, T).float(), dtype=torch.bfloat16)
    rows = 512
    xt = x[:rows].double().reshape(rows // T, T, K // T, T).permute(0, 2, 1, 3).reshape(rows // T, K // T, T * T)
    u = xt @ snf.e_x.double().T                                    # (bi, bk, r)
    prod = torch.einsum("ikp,pjk->ijp", u, w.double())              # (bi, bj, r)
    yt = prod @ snf.d.double()                                     # (bi, bj, 16)
    yref = yt.reshape(rows // T, N // T, T, T).permute(0, 2, 1, 3).reshape(rows, N)
    for name, prod in (("F24", "f24"), ("auto", None), ("fp32", torch.float32)):
        try:
            y = _forward(x, w, snf, products=prod)
        except ValueError:
            continue
        err = float((y[:rows].double() - yref).norm() / yref.norm())
        for _ in range(3):
            _forward(x, w, snf, products=prod)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            _forward(x, w, snf, products=prod)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"shape": [M, K, N], "r": R, "products": name, "rel_err": err,
                          "ms": e0.elapsed_time(e1) / 20}))
