"""Per-launch spans of the 8192^3 forward (and the config-2 layer step) from the probe
library's globaltimer trace (STL_TRACE=1): each kernel's [first CTA entry, last CTA exit] and
the gaps between consecutive launches. One JSON line per pipeline."""
import ctypes
import json
import os
import sys

os.environ.setdefault("STL_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_12211_b200 import _lib  # noqa: E402
os.environ.setdefault("STL_LIB", str(_lib.PROBE_LIB_PATH))
import torch  # noqa: E402
import paper_2503_12211_b200 as stl  # noqa: E402

lib = _lib.load()
lib.stl_trace_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
dev = torch.device("cuda")
T, R = 4, 24
s = torch.cuda.current_stream().cuda_stream


def spans(names, fn, reps=6):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    lib.stl_trace_reset()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (2 * 4096))()
    k = lib.stl_trace_read(buf, 4096)
    sp = [(buf[2 * i], buf[2 * i + 1]) for i in range(k)]
    per = len(names)
    rows = []
    for r in range(1, reps):  # skip the first (cold) repetition
        seq = sp[r * per:(r + 1) * per]
        prev_end = sp[r * per - 1][1]
        row = {}
        for nm, (a, b) in zip(names, seq):
            row[nm] = {"gap_us": round((a - prev_end) / 1e3, 1), "span_us": round((b - a) / 1e3, 1)}
            prev_end = b
        row["total_us"] = round((seq[-1][1] - sp[r * per - 1][1]) / 1e3, 1)
        rows.append(row)
    return rows


n = 8192
b = n // T
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
xf = torch.randn((n, n), device=dev).to(torch.bfloat16)
wf = (torch.randn((R, b, b), device=dev) * 0.02).to(torch.bfloat16)
uf = torch.empty((R, b, b), dtype=torch.bfloat16, device=dev)
sb = int(lib.stl_forward_scratch_bytes(n, n, n, T, R, _lib.STL_BF16))
sf = torch.empty((sb,), dtype=torch.uint8, device=dev)
yf = torch.empty((n, n), dtype=torch.bfloat16, device=dev)


def fwd():
    _lib.check(lib.stl_forward(xf.data_ptr(), n, n, n, wf.data_ptr(), n, snf.e_x.data_ptr(),
                               snf.d.data_ptr(), T, R, _lib.STL_BF16, yf.data_ptr(), n,
                               uf.data_ptr(), None, sf.data_ptr(), sb, s))


for row in spans(["encode", "gemm", "decode"], fwd):
    print(json.dumps({"fwd8192": row}), flush=True)

# per-CTA stamps of the traced forwards' transforms, relative to the predecessor's last exit
lib.stl_trace_read_cta.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int, ctypes.c_int]
lib.stl_trace_reset()
for _ in range(4):
    fwd()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (2 * 4096))()
k = lib.stl_trace_read(buf, 4096)
grid = torch.cuda.get_device_properties(0).multi_processor_count
cta = (ctypes.c_ulonglong * (grid * 4))()
for slot in (3 * 2, 3 * 2 + 2, 3 * 3, 3 * 3 + 2):  # encode / decode of forwards 2 and 3
    lib.stl_trace_read_cta(cta, slot, grid)
    pred_end = buf[2 * (slot - 1) + 1]
    rel = [[(cta[4 * c + e] - pred_end) / 1e3 for e in range(4)] for c in range(grid)]
    out = {}
    for e, nm in enumerate(("entry", "after_griddep", "first_data", "loop_end")):
        v = sorted(r[e] for r in rel)
        out[nm] = [round(v[0], 1), round(v[len(v) // 2], 1), round(v[-1], 1)]
    print(json.dumps({"slot": slot, "kernel": "encode" if slot % 3 == 0 else "decode",
                      "us_after_predecessor_end_min_med_max": out}), flush=True)

# which CTAs straggle? (encode of forward 3: blockIdx -> loop end after the predecessor's end)
if os.environ.get("TRACE_CTA_DUMP"):
    lib.stl_trace_read_cta(cta, 9, grid)
    pred_end = buf[2 * 8 + 1]
    ends = sorted(((cta[4 * c + 3] - pred_end) / 1e3, c) for c in range(grid))
    print(json.dumps({"encode_loop_end_latest": [(round(t, 1), c) for t, c in ends[-12:]],
                      "earliest": [(round(t, 1), c) for t, c in ends[:6]]}), flush=True)
    lib.stl_trace_read_cta(cta, 11, grid)
    pred_end = buf[2 * 10 + 1]
    ends = sorted(((cta[4 * c + 3] - pred_end) / 1e3, c) for c in range(grid))
    print(json.dumps({"decode_loop_end_latest": [(round(t, 1), c) for t, c in ends[-12:]],
                      "earliest": [(round(t, 1), c) for t, c in ends[:6]]}), flush=True)
