"""Streaming-transform tuning probe (probe library; STL_STREAM_* switches from the environment):
8192^3 t=4 r=24 bf16 encode and decode alone, and the whole forward, CUDA-event timed.
Prints one JSON line incl. hashes of the outputs (scheduling switches must not change them)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_12211_b200 import _lib  # noqa: E402
import paper_2503_12211_b200 as stl  # noqa: E402

os.environ.setdefault("STL_LIB", str(_lib.PROBE_LIB_PATH))
lib = _lib.load()
dev = torch.device("cuda")
T, R, n = 4, 24, 8192
b = n // T
torch.manual_seed(0)
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
wf = stl.weights_to_planes(stl.encode_tiles(torch.randn((n, n), device=dev) / n ** 0.5, snf.e_w, T),
                           dtype=torch.bfloat16)
xf = torch.randn((n, n), device=dev).to(torch.bfloat16)
uf = torch.empty((R, b, b), dtype=torch.bfloat16, device=dev)
ye = torch.randn((R, b, b), device=dev).to(torch.bfloat16)
sf = torch.empty((int(lib.stl_forward_scratch_bytes(n, n, n, T, R, _lib.STL_BF16)),), dtype=torch.uint8,
                 device=dev)
yf = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
y2 = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
s = torch.cuda.current_stream().cuda_stream


def fwd():
    _lib.check(lib.stl_forward(xf.data_ptr(), n, n, n, wf.data_ptr(), n, snf.e_x.data_ptr(),
                               snf.d.data_ptr(), T, R, _lib.STL_BF16, yf.data_ptr(), n,
                               uf.data_ptr(), None, sf.data_ptr(), sf.numel(), s))


def enc():
    _lib.check(lib.stl_encode(xf.data_ptr(), 1, n, n, n, snf.e_x.data_ptr(), T, R, uf.data_ptr(), 1, s))


def dec():
    _lib.check(lib.stl_decode(ye.data_ptr(), 1, b, b, R, snf.d.data_ptr(), T, y2.data_ptr(), 1, n, s))


def timed(fn, k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def h(t):
    return hashlib.sha256(t.view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:12]


for _ in range(3):
    fwd(); enc(); dec()
res = {k: v for k, v in os.environ.items() if k.startswith("STL_")}
out = {}
for name, fn in (("enc", enc), ("dec", dec), ("fwd", fwd)):
    ts = [timed(fn, 10) for _ in range(5)]
    out[name + "_us"] = round(min(ts) * 1e3, 1)
    out[name + "_med_us"] = round(sorted(ts)[2] * 1e3, 1)
res.update(out)
lib.stl_profile_enable(1)
lib.stl_profile_reset()
for _ in range(10):
    fwd()
torch.cuda.synchronize()
recs = _lib.profile_records()
lib.stl_profile_enable(0)
res["fwd_parts_us"] = {nm: round(ms / 10 * 1e3, 1) for nm, ms, _ in recs}
enc(); dec(); fwd()
torch.cuda.synchronize()
res["h"] = [h(uf), h(y2), h(yf)]
print(json.dumps(res), flush=True)
