"""Interleaved A/B of probe-build switches (STL_LIB = libstl_b200_probe.so): every round runs
each variant once (a few back-to-back calls, CUDA events) so clock / power drift hits all
variants alike; prints per-variant medians. VARIANTS="NAME=ENV,ENV;NAME2=..." (ENV = K=V)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200.layer import LayerCache, backward_raw  # noqa: E402
from paper_2503_12211_b200.snf_operator import _forward  # noqa: E402

assert "probe" in os.environ.get("STL_LIB", ""), "run with STL_LIB=<probe library>"
dev = torch.device("cuda")
T, R = 4, 24
stl.set_check_finite(False)


def problem(M, K, N):
    snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
    g = torch.Generator(device=dev).manual_seed(1)
    x = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn((R, N // T, K // T), device=dev, generator=g) * 0.03).to(torch.bfloat16)
    gy = torch.randn((M, N), device=dev, generator=g).to(torch.bfloat16)
    return snf, x, w, gy


work = {}
snf8, x8, w8, _ = problem(8192, 8192, 8192)
work["fwd8192"] = lambda: _forward(x8, w8, snf8)
snf2, x2, w2, gy2 = problem(8192, 4096, 4096)
work["fwd_cfg2"] = lambda: _forward(x2, w2, snf2)


def step_cfg2():
    y, u, ye = _forward(x2, w2, snf2, keep_cache=True)
    backward_raw(snf2, w2, LayerCache(x2, u, ye), gy2)


work["step_cfg2"] = step_cfg2
from paper_2503_12211_b200 import _lib  # noqa: E402

ga = torch.randn((R, 2048, 2048), device=dev).to(torch.bfloat16)
gb = torch.randn((R, 2048, 2048), device=dev).to(torch.bfloat16)
gc = torch.empty((R, 2048, 2048), device=dev, dtype=torch.bfloat16)
work["gemm8192"] = lambda: _lib.check(_lib.load().stl_slice_gemm(
    ga.data_ptr(), 0, gb.data_ptr(), 0, gc.data_ptr(), 1, 1, R, 2048, 2048, 2048,
    torch.cuda.current_stream().cuda_stream))
a = torch.randn((8192, 8192), device=dev).to(torch.bfloat16)
work["cublas8192"] = lambda: a @ a

only = os.environ.get("WORK")
if only:
    work = {k: v for k, v in work.items() if k in only.split(",")}
variants = {}
for part in os.environ.get("VARIANTS", "base=").split(";"):
    name, _, envs = part.partition("=")
    variants[name] = dict(kv.split(":", 1) for kv in envs.split(",") if kv)
keys = set(k for v in variants.values() for k in v)
rounds, reps = int(os.environ.get("ROUNDS", "15")), int(os.environ.get("REPS", "5"))
res = {(v, w): [] for v in variants for w in work}
for r in range(rounds):
    for vname, env in variants.items():
        for k in keys:
            os.environ.pop(k, None)
        os.environ.update(env)
        for wname, fn in work.items():
            if wname == "cublas8192" and vname != next(iter(variants)):
                continue
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            if r > 0:
                res[(vname, wname)].append(e0.elapsed_time(e1) / reps)
out = {f"{v}/{w}": round(statistics.median(t), 4) for (v, w), t in res.items() if t}
print(json.dumps(out))
