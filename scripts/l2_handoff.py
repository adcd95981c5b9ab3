"""8192^3 bf16 STL forward (t=4, r=24) timed like bench.py's north-star leg, for the L2-handoff
budget given by STL_L2_KEEP_MB (probe library). Prints one JSON line incl. a hash of y (the
handoff changes cache policies only: y must be bit-identical for every budget)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_12211_b200 import _lib  # noqa: E402
import paper_2503_12211_b200 as stl  # noqa: E402

lib = _lib.load(_lib.PROBE_LIB_PATH)
dev = torch.device("cuda")
T, R, n = 4, 24, 8192
torch.manual_seed(0)
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
wf = stl.weights_to_planes(stl.encode_tiles(torch.randn((n, n), device=dev) / n ** 0.5, snf.e_w, T),
                           dtype=torch.bfloat16)
xf = torch.randn((n, n), device=dev).to(torch.bfloat16)
uf = torch.empty((R, n // T, n // T), dtype=torch.bfloat16, device=dev)
sf = torch.empty((int(lib.stl_forward_scratch_bytes(n, n, n, T, R, _lib.STL_BF16)),), dtype=torch.uint8,
                 device=dev)
yf = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
wdf = torch.randn((n, n), device=dev).to(torch.bfloat16)
ydf = torch.empty((n, n), device=dev, dtype=torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream


def fwd():
    _lib.check(lib.stl_forward(xf.data_ptr(), n, n, n, wf.data_ptr(), n, snf.e_x.data_ptr(),
                               snf.d.data_ptr(), T, R, _lib.STL_BF16, yf.data_ptr(), n,
                               uf.data_ptr(), None, sf.data_ptr(), sf.numel(), s))


def timed(fn, k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


for _ in range(5):
    fwd()
    torch.matmul(xf, wdf, out=ydf)
res = {k: v for k, v in os.environ.items() if k.startswith("STL_L2")}
st, cb = [], []
for rep in range(5):
    st.append(timed(fwd, 20))
    cb.append(timed(lambda: torch.matmul(xf, wdf, out=ydf), 20))
fwd()
torch.cuda.synchronize()
res["stl_ms"] = sorted(st)[2]
res["stl_min"] = min(st)
res["cublas_min"] = None
res["stl_all"] = [round(v, 4) for v in st]
res["cublas_ms"] = sorted(cb)[2]
res["cublas_min"] = min(cb)
res["speedup"] = res["cublas_ms"] / res["stl_ms"]
res["y_sha"] = hashlib.sha256(yf.view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:16]
ref = (xf.float() @ torch.eye(1, device=dev).expand(1, 1)) if False else None
print(json.dumps(res), flush=True)
