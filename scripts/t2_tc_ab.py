"""t = 2 transforms at 8192^2 (r = 16 / 24 / 32): encode, decode alone and the forward, CUDA-event
timed (probe library; STL_T2_TC=0 selects the register-streaming kernels). One JSON line per r."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_12211_b200 import _lib  # noqa: E402
os.environ.setdefault("STL_LIB", str(_lib.PROBE_LIB_PATH))
import torch  # noqa: E402
import paper_2503_12211_b200 as stl  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda")
T, n = 2, 8192
b = n // T
s = torch.cuda.current_stream().cuda_stream


def timed(fn, k=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / k * 1e3)
    return round(sorted(ts)[2], 1)


x = torch.randn((n, n), device=dev).to(torch.bfloat16)
y = torch.empty((n, n), device=dev, dtype=torch.bfloat16)
for R in (16, 24, 32):
    snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
    u = torch.empty((R, b, b), dtype=torch.bfloat16, device=dev)
    ye = torch.randn((R, b, b), device=dev).to(torch.bfloat16)
    w = (torch.randn((R, b, b), device=dev) * 0.02).to(torch.bfloat16)
    sb = int(lib.stl_forward_scratch_bytes(n, n, n, T, R, _lib.STL_BF16))
    sf = torch.empty((sb,), dtype=torch.uint8, device=dev)

    def enc():
        _lib.check(lib.stl_encode(x.data_ptr(), 1, n, n, n, snf.e_x.data_ptr(), T, R, u.data_ptr(), 1, s))

    def dec():
        _lib.check(lib.stl_decode(ye.data_ptr(), 1, b, b, R, snf.d.data_ptr(), T, y.data_ptr(), 1, n, s))

    def fwd():
        _lib.check(lib.stl_forward(x.data_ptr(), n, n, n, w.data_ptr(), n, snf.e_x.data_ptr(),
                                   snf.d.data_ptr(), T, R, _lib.STL_BF16, y.data_ptr(), n,
                                   u.data_ptr(), None, sf.data_ptr(), sb, s))

    nbytes = n * n * 2 + R * b * b * 2
    te, td = timed(enc), timed(dec)
    print(json.dumps({"STL_T2_TC": os.environ.get("STL_T2_TC", "1"), "r": R, "enc_us": te, "dec_us": td,
                      "enc_hbm_frac": round(nbytes / te / 1e3 / 6553.6, 3),
                      "dec_hbm_frac": round(nbytes / td / 1e3 / 6553.6, 3),
                      "fwd_us": timed(fwd, 3)}), flush=True)
