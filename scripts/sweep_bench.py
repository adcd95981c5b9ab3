"""Run bench.py's configs[2] rank sweep alone (one JSON line per point)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
lib = _lib.load()
stream = torch.cuda.current_stream().cuda_stream
peaks = bench.load_peaks() if hasattr(bench, "load_peaks") else None


def timed(fn, steps, profile=False):
    torch.cuda.synchronize()
    if profile:
        lib.stl_profile_reset()
        lib.stl_profile_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    if profile:
        lib.stl_profile_enable(0)
    return e0.elapsed_time(e1)


for pt in bench.rank_sweep(stl, lib, _lib, dev, stream, peaks, timed):
    print(json.dumps(pt), flush=True)
