"""Time the STL forward (stl_forward) at config-2 and 8192^3 shapes, fused vs unfused."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_12211_b200 as stl
from paper_2503_12211_b200 import _lib
lib = _lib.load()
dev = torch.device("cuda")
T, R = 4, int(os.environ.get("R", "24"))
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
for (M, K, N) in ((8192, 4096, 4096), (8192, 8192, 8192)):
    x = torch.randn((M, K), device=dev).to(torch.bfloat16)
    w = torch.randn((R, N // T, K // T), device=dev).to(torch.bfloat16)
    u = torch.empty((R, M // T, K // T), device=dev, dtype=torch.bfloat16)
    y = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
    for fused in (1, 0):
        lib.stl_set_fusion(fused)
        sc = torch.empty((int(lib.stl_forward_scratch_bytes(M, K, N, T, R, 1)),), dtype=torch.uint8, device=dev)
        s = torch.cuda.current_stream().cuda_stream
        def run():
            _lib.check(lib.stl_forward(x.data_ptr(), M, K, K, w.data_ptr(), N, snf.e_x.data_ptr(), snf.d.data_ptr(),
                                       T, R, 1, y.data_ptr(), N, u.data_ptr(), None, sc.data_ptr(), sc.numel(), s))
        for _ in range(3): run()
        torch.cuda.synchronize()
        lib.stl_profile_reset(); lib.stl_profile_enable(1)
        n = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): run()
        e1.record(); torch.cuda.synchronize(); lib.stl_profile_enable(0)
        agg = {}
        for name, ms, _ in _lib.profile_records():
            agg[name] = agg.get(name, 0) + ms / n
        print(json.dumps({"M": M, "K": K, "N": N, "r": R, "fused": fused, "ms": e0.elapsed_time(e1) / n,
                          "kernels": {k: round(v, 4) for k, v in agg.items()},
                          "pairs_env": os.environ.get("STL_FUSED_PAIRS")}))
