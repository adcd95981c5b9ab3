"""f1: a 3-layer bf16 STL chain at 8192^3 (t=4, r=24) kept in encoded space (Algorithm 2,
snf_operator.py:175-188) against the same 3 layers run as separate forwards (encode ->
slice GEMMs -> decode each), CUDA-event timed, plus the reference cost model's IO
(io_fused_chain vs layers * io_square, cost_model.py:94-124). One JSON line."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200 import _lib  # noqa: E402


def chain_bench(n=8192, t=4, r=24, layers=3, iters=3):
    lib = _lib.load()
    dev = torch.device("cuda")
    s = torch.cuda.current_stream().cuda_stream
    bf = torch.bfloat16
    b = n // t
    snf = stl.random_gaussian_init(t, r, stl.make_rng(0), scale=0.5).to(dev)
    ws = [(torch.randn((r, b, b), device=dev) * 0.02).to(bf) for _ in range(layers)]
    x = torch.randn((n, n), device=dev).to(bf)
    ys = [torch.empty((n, n), device=dev, dtype=bf) for _ in range(layers)]
    u = torch.empty((r, b, b), device=dev, dtype=bf)
    sb = int(lib.stl_forward_scratch_bytes(n, n, n, t, r, _lib.STL_BF16))
    scratch = torch.empty((sb,), dtype=torch.uint8, device=dev)
    h = [torch.empty((r, b, b), device=dev, dtype=bf) for _ in range(2)]
    mixed = torch.empty((r, b, b), device=dev, dtype=bf)
    comp = torch.empty((r, r), device=dev)
    yf = torch.empty((n, n), device=dev, dtype=bf)

    def unfused():
        inp = x
        for i in range(layers):
            _lib.check(lib.stl_forward(inp.data_ptr(), n, n, n, ws[i].data_ptr(), n,
                                       snf.e_x.data_ptr(), snf.d.data_ptr(), t, r, _lib.STL_BF16,
                                       ys[i].data_ptr(), n, u.data_ptr(), None, scratch.data_ptr(),
                                       sb, s))
            inp = ys[i]

    def fused():
        _lib.check(lib.stl_encode(x.data_ptr(), _lib.STL_BF16, n, n, n, snf.e_x.data_ptr(), t, r,
                                  u.data_ptr(), _lib.STL_BF16, s))
        _lib.check(lib.stl_slice_gemm(u.data_ptr(), 0, ws[0].data_ptr(), 0, h[0].data_ptr(),
                                      _lib.STL_BF16, _lib.STL_BF16, r, b, b, b, s))
        for i in range(1, layers):
            _lib.check(lib.stl_fused_step_ex(h[(i - 1) % 2].data_ptr(), _lib.STL_BF16, b, b,
                                             ws[i].data_ptr(), b, snf.e_x.data_ptr(),
                                             snf.d.data_ptr(), t, r, _lib.STL_BF16,
                                             h[i % 2].data_ptr(), _lib.STL_BF16, mixed.data_ptr(),
                                             comp.data_ptr(), s))
        _lib.check(lib.stl_decode(h[(layers - 1) % 2].data_ptr(), _lib.STL_BF16, b, b, r,
                                  snf.d.data_ptr(), t, yf.data_ptr(), _lib.STL_BF16, n, s))

    def timed(fn, k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    # alternating short blocks after idle (both at unthrottled clocks, like bench.py's north
    # star), medians
    for _ in range(3):
        unfused()
        fused()
    ub, fb = [], []
    for _ in range(7):
        time.sleep(0.06)
        ub.append(timed(unfused, iters))
        time.sleep(0.06)
        fb.append(timed(fused, iters))
    u_ms, f_ms = statistics.median(ub), statistics.median(fb)
    unfused()
    fused()
    torch.cuda.synchronize()
    err = ((yf.float() - ys[-1].float()).norm() / ys[-1].float().norm()).item()
    lib.stl_profile_reset()
    lib.stl_profile_enable(1)
    fused()
    torch.cuda.synchronize()
    lib.stl_profile_enable(0)
    remix = [ms for nm, ms, _ in _lib.profile_records() if nm == "remix"]
    remix_us = 1e3 * sum(remix) / max(len(remix), 1)
    remix_bytes = 2 * r * b * b * 2
    io_l = stl.io_square(n, t, r, 2)
    io_chain = stl.io_fused_chain(n, t, r, layers, 2)
    return {"n": n, "t": t, "r": r, "layers": layers, "dtype": "bf16",
            "timing": f"7 alternating blocks of {iters} chains (separate forwards, fused), each "
                      "after 60 ms idle, medians",
            "unfused_ms": u_ms, "fused_chain_ms": f_ms, "speedup": u_ms / f_ms,
            "rel_diff_fused_vs_unfused": err,
            "remix_us": remix_us, "remix_GBs": remix_bytes / (remix_us * 1e-6) / 1e9,
            "cost_model_io_unfused": layers * (io_l[0] if isinstance(io_l, tuple) else io_l),
            "cost_model_io_fused_chain": io_chain}


if __name__ == "__main__":
    print(json.dumps(chain_bench()), flush=True)
