"""Co-residency probe (probe library): can the 8192^3 forward's encode / decode run beside the
slice GEMM on the same SMs without slowing it?

Runs the three forward kernels alone and pairwise on two streams over INDEPENDENT buffers (no
data dependence; this measures interference only). Configure with the probe switches:
  STL_GEMM_STAGES=4          4-stage GEMM ring (161.5 KB smem) so a transform CTA fits beside it
  STL_STREAM_CW=8            8 consumer warps per transform CTA (288 threads)
  STL_STREAM_SMEM_KB=60      transform CTA shared-memory budget
Prints one JSON line.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_12211_b200 import _lib  # noqa: E402

lib = _lib.load(_lib.PROBE_LIB_PATH)
dev = torch.device("cuda")
T, R, n = 4, 24, 8192
b = n // T
bf = torch.bfloat16
g = torch.Generator(device=dev).manual_seed(0)
X = torch.randn((n, n), device=dev, generator=g).to(bf)
X2 = torch.randn((n, n), device=dev, generator=g).to(bf)
Xe = torch.empty((R, b, b), device=dev, dtype=bf)
Xe2 = torch.empty((R, b, b), device=dev, dtype=bf)
W = (torch.randn((R, b, b), device=dev, generator=g) * 0.02).to(bf)
Ye = torch.empty((R, b, b), device=dev, dtype=bf)
Ye2 = (torch.randn((R, b, b), device=dev, generator=g)).to(bf)
Y = torch.empty((n, n), device=dev, dtype=bf)
ex = torch.randn((R, 16), device=dev, generator=g) * 0.5
dd = torch.randn((R, 16), device=dev, generator=g) * 0.5


def enc(s, x=X2, xe=Xe2):
    _lib.check(lib.stl_encode(x.data_ptr(), 1, n, n, n, ex.data_ptr(), T, R, xe.data_ptr(), 1,
                              s.cuda_stream))


def gemm(s):
    _lib.check(lib.stl_slice_gemm(Xe.data_ptr(), 0, W.data_ptr(), 0, Ye.data_ptr(), 1, 1, R, b, b, b,
                                  s.cuda_stream))


def dec(s):
    _lib.check(lib.stl_decode(Ye2.data_ptr(), 1, b, b, R, dd.data_ptr(), T, Y.data_ptr(), 1, n,
                              s.cuda_stream))


s0 = torch.cuda.current_stream()
s1 = torch.cuda.Stream()
s2 = torch.cuda.Stream()


def timed(fns, reps=10, warm=3):
    """fns: list of (fn) launched on streams s1, s2, ... concurrently; returns median ms of the
    joined region and of each stream."""
    streams = [s1, s2][: len(fns)]
    tot, per = [], [[] for _ in fns]
    for it in range(warm + reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(s0)
        ends = []
        for f, st in zip(fns, streams):
            st.wait_event(e0)
            f(st)
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            ends.append(e)
        for e in ends:
            s0.wait_event(e)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(s0)
        torch.cuda.synchronize()
        if it >= warm:
            tot.append(e0.elapsed_time(e1))
            for i, e in enumerate(ends):
                per[i].append(e0.elapsed_time(e))
    med = lambda v: sorted(v)[len(v) // 2]
    return round(med(tot) * 1000, 1), [round(med(p) * 1000, 1) for p in per]


enc(s0, X, Xe)  # real operands for the GEMM
torch.cuda.synchronize()
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("STL_")}}
out["gemm_us"] = timed([gemm])[0]
out["enc_us"] = timed([enc])[0]
out["dec_us"] = timed([dec])[0]
out["gemm||enc"] = timed([gemm, enc])
out["enc||gemm"] = timed([enc, gemm])
out["gemm||dec"] = timed([gemm, dec])
out["seq_gemm_enc_dec_us"] = round(out["gemm_us"] + out["enc_us"] + out["dec_us"], 1)
print(json.dumps(out))
