"""cuBLAS batched GEMM on the STL slice shapes (reference point for the tcgen05 slice GEMM)."""
import json, torch
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for name, (r, M, N, K) in {"cfg2_fwd": (24, 2048, 1024, 1024), "cfg2_gw": (24, 1024, 1024, 2048), "n8192": (24, 2048, 2048, 2048)}.items():
    a = torch.randn(r, M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(r, K, N, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(r, M, N, device="cuda", dtype=torch.bfloat16)
    ms = t(lambda: torch.bmm(a, b, out=c))
    print(json.dumps({"shape": name, "cublas_bmm_bf16out_ms": ms, "tflops": 2 * r * M * N * K / ms / 1e9}))
