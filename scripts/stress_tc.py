"""Stress of the tcgen05 transforms' protocols (stage ring, TMEM double buffer, unit ring, the
dynamic-tail counter): many back-to-back config-2 steps, 8192^3 forwards and fused-chain steps,
every output compared bit for bit with the first run's every `CHECK` iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_12211_b200 as stl  # noqa: E402
from paper_2503_12211_b200.layer import LayerCache, backward_raw  # noqa: E402
from paper_2503_12211_b200.snf_operator import _forward  # noqa: E402

dev = torch.device("cuda")
CHECK = int(os.environ.get("CHECK", "25"))
T, R = 4, 24
snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
g = torch.Generator(device=dev).manual_seed(7)


def run(name, fn, iters):
    ref = [o.clone() for o in fn()]
    bad = 0
    for i in range(iters):
        out = fn()
        if (i + 1) % CHECK == 0:
            for a, b in zip(out, ref):
                if not torch.equal(a, b):
                    bad += 1
    torch.cuda.synchronize()
    print(f"{name}: {iters} iterations, {bad} mismatching checks", flush=True)
    return bad


M, K, N = 8192, 4096, 4096
w = (torch.randn((R, N // T, K // T), device=dev, generator=g) * 0.03).to(torch.bfloat16)
x = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
gy = torch.randn((M, N), device=dev, generator=g).to(torch.bfloat16)


def step():
    y, u, ye = _forward(x, w, snf, keep_cache=True)
    return [y] + list(backward_raw(snf, w, LayerCache(x, u, ye), gy))


n = 8192
w8 = (torch.randn((R, n // T, n // T), device=dev, generator=g) * 0.02).to(torch.bfloat16)
x8 = torch.randn((n, n), device=dev, generator=g).to(torch.bfloat16)


def fwd8():
    return [_forward(x8, w8, snf)]


w8v = w8.permute(1, 2, 0)  # the (I, J, r) view of the planes
h0 = stl._slice_products(stl.encode_tiles(x8, snf.e_x, T), w8v).to(torch.bfloat16)


def chain():
    return [stl.stl_fused_step(h0, w8v, snf)]


bad = run("config-2 step", step, int(os.environ.get("STEPS", "1000")))
bad += run("8192^3 forward", fwd8, int(os.environ.get("FWDS", "600")))
bad += run("fused-chain step", chain, int(os.environ.get("CHAINS", "300")))
print("stress", "ok" if bad == 0 else f"FAILED ({bad})")
