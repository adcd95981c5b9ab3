"""Why are the transforms slower inside the forward than alone? Times the 8192^3 decode (and
encode) right after different predecessors (events between launches):
  same      : after itself (the standalone loop)
  gemm      : after the forward's slice GEMM (dirty slice products in L2)
  dirty     : after a 96 MB memset (dirty lines, no tensor work)
  clean     : after a 400 MB read-only reduction (L2 full of clean lines)
  idle      : after a 50 us sleep kernel
One JSON line (medians over 20 pairs)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_12211_b200 import _lib  # noqa: E402
import paper_2503_12211_b200 as stl  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda")
T, R, n = 4, 24, 8192
b = n // T
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
x = torch.randn((n, n), device=dev).to(torch.bfloat16)
u = torch.empty((R, b, b), dtype=torch.bfloat16, device=dev)
w = (torch.randn((R, b, b), device=dev) * 0.02).to(torch.bfloat16)
ye = torch.empty((R, b, b), dtype=torch.bfloat16, device=dev)
y = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
dirty = torch.empty((96 << 20,), dtype=torch.uint8, device=dev)
big = torch.randn((100 << 20,), device=dev)
s = torch.cuda.current_stream().cuda_stream


def enc():
    _lib.check(lib.stl_encode(x.data_ptr(), 1, n, n, n, snf.e_x.data_ptr(), T, R, u.data_ptr(), 1, s))


def gemm():
    _lib.check(lib.stl_slice_gemm(u.data_ptr(), 0, w.data_ptr(), 0, ye.data_ptr(), 1, 1, R, b, b, b, s))


def dec():
    _lib.check(lib.stl_decode(ye.data_ptr(), 1, b, b, R, snf.d.data_ptr(), T, y.data_ptr(), 1, n, s))


preds = {"same": None, "gemm": gemm, "dirty": lambda: dirty.fill_(1),
         "clean": lambda: big.sum(), "idle": lambda: torch.cuda._sleep(100000),
         "enc": enc}
enc(); gemm(); dec()
torch.cuda.synchronize()
out = {}
for target_name, target in (("dec", dec), ("enc", enc)):
    for pname, pred in preds.items():
        ts = []
        for _ in range(20):
            if pred is not None:
                pred()
            else:
                target()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            target()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        out[f"{target_name}_after_{pname}_us"] = round(sorted(ts)[10], 1)
print(json.dumps(out), flush=True)
