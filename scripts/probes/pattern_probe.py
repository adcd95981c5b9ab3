"""Data-movement floor of the streaming transforms at 8192^3 (t=4, r=24): encode-like (4 matrix
rows in, 24 plane segments out) and decode-like (the reverse) bulk-copy pipelines for several
unit sizes, next to a contiguous copy. Measurement aid; prints JSON lines."""
import ctypes
import json
import os
import subprocess
import sys

import torch

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "libpattern.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", "-o", so, os.path.join(here, "pattern_probe.cu")])
lib = ctypes.CDLL(so)
lib.probe_pattern.argtypes = [ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_int, ctypes.c_int] + \
    [ctypes.c_int64] * 4 + [ctypes.c_int, ctypes.c_int] + [ctypes.c_int64] * 4 + \
    [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
n, r = 8192, 24
b = n // 4
X = torch.empty(n * n * 2, dtype=torch.uint8, device="cuda")
P = torch.empty(r * b * b * 2, dtype=torch.uint8, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count


def run(name, src, dst, pin, pout, nunits, grid, nst, total_bytes):
    args = [src.data_ptr(), dst.data_ptr(), *pin, *pout, nunits, grid, nst, None]
    for _ in range(3):
        assert lib.probe_pattern(*args) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record()
        lib.probe_pattern(*args)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(json.dumps({"case": name, "grid": grid, "nst": nst, "us": round(ms * 1e3, 1),
                      "GBs": round(total_bytes / ms / 1e6, 1)}), flush=True)


# planes -> planes (the fused-chain remix): 24 segments in, 24 out per unit
if os.environ.get("PP_REMIX"):  # only these cases
    P2 = torch.empty_like(P)
    for U in (512, 1024):
        planes = (1, r, U * 2, 0, 0, b * b * 2)
        nunits = b * (b // U)
        for grid_mult, nst in ((1, 4), (2, 2), (2, 3), (1, 8)):
            try:
                run(f"remix U={U}", P, P2, planes, planes, nunits, sms * grid_mult, nst, 2 * r * b * b * 2)
            except AssertionError:
                pass
    sys.exit(0)


tot = n * n * 2 + r * b * b * 2
for U in (128, 256, 512, 1024, 2048):
    upr = b // U
    rows = (0, 4, U * 8, upr, n * 2, 0)
    planes = (1, r, U * 2, 0, 0, b * b * 2)
    nunits = b * upr
    stage = max(4 * U * 8, r * U * 2)
    for grid_mult in (1, 2):
        nst_max = (220 * 1024 // grid_mult) // ((stage + 1023) // 1024 * 1024)
        for nst in sorted({2, 4, min(8, nst_max), min(16, nst_max)}):
            if nst < 2 or nst > 16 or nst > nst_max:
                continue
            run(f"encode U={U}", X, P, rows, planes, nunits, sms * grid_mult, nst, tot)
            run(f"decode U={U}", P, X, planes, rows, nunits, sms * grid_mult, nst, tot)
# contiguous copy of the same byte count (read 1 GiB... here: planes -> planes)
for ch in (16384, 32768):
    nunits = (r * b * b * 2) // ch
    pl = (1, 1, ch, 0, 0, 0)
    for nst in (4, 6):
        run(f"copy chunk={ch}", P, torch.empty_like(P), pl, pl, nunits, sms, nst, 2 * r * b * b * 2)
for U in (512, 1024):  # writes only / reads only (rows vs planes)
    upr = b // U
    rows = (0, 4, U * 8, upr, n * 2, 0)
    planes = (1, r, U * 2, 0, 0, b * b * 2)
    none_out = (1, 0, 0, 0, 0, 0)
    run(f"read rows U={U}", X, P, rows, none_out, b * upr, sms, 8, n * n * 2)
    run(f"read planes U={U}", P, X, planes, none_out, b * upr, sms, 8, r * b * b * 2)
