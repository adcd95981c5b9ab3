"""Per-kernel times of the config-2 layer step with the mma vs FFMA transforms."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_12211_b200 as stl
from paper_2503_12211_b200 import _lib
from paper_2503_12211_b200.layer import backward_raw
lib = _lib.load()
dev = torch.device("cuda")
T, R, M, K, N = 4, 24, 8192, 4096, 4096
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
w = torch.randn((R, N // T, K // T), device=dev).to(torch.bfloat16) * 0.03
x = torch.randn((M, K), device=dev).to(torch.bfloat16)
gy = torch.randn((M, N), device=dev).to(torch.bfloat16)
layer_snf = snf
for mode in (int(os.environ.get("STL_FUSION_BITS", "0")),):
    lib.stl_set_fusion(mode)
    def step():
        from paper_2503_12211_b200.snf_operator import _forward
        from paper_2503_12211_b200.layer import LayerCache
        y, u, ye = _forward(x, w, layer_snf, keep_cache=True)
        backward_raw(layer_snf, w, LayerCache(x, u, ye), gy)
    for _ in range(3): step()
    torch.cuda.synchronize()
    lib.stl_profile_reset(); lib.stl_profile_enable(1)
    n = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): step()
    e1.record(); torch.cuda.synchronize(); lib.stl_profile_enable(0)
    agg = {}
    for name, ms, _ in _lib.profile_records():
        agg[name] = agg.get(name, 0) + ms / n
    print(json.dumps({"mode": mode, "fused": mode & 1, "ffma": (mode >> 1) & 1,
                      "ms_step": e0.elapsed_time(e1) / n, "kernels_ms": {k: round(v, 4) for k, v in agg.items()}}))
lib.stl_set_fusion(0)
