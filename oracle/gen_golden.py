"""Generate golden vectors for the STL hot path by running the REFERENCE itself.

Run in the build container (where /root/reference is mounted):

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Writes tests/golden/*.npz. Every case stores its seeded inputs and the reference's outputs,
computed by strassen_tile's own functions (encode_tiles, decode_tiles, _slice_products,
stl_batched, stl_reference, stl_fused_step, _layer_forward_cached, _layer_backward,
strassen_rank49, random_gaussian_init, cost_model). The GPU box never reads /root/reference:
tests compare against these committed fixtures.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, str(REF))
    import strassen_tile as st
    from strassen_tile import cost_model, snf_operator, strassen_basis, toy_network

    OUT.mkdir(parents=True, exist_ok=True)
    rng = st.make_rng(20260317)

    # 1. encode / decode / slice products / batched / loop reference over a (t, r, shape) grid
    cases = {}
    idx = 0
    for t in (1, 2, 4):
        for (bi, bk, bj) in ((1, 1, 1), (2, 3, 2), (3, 2, 5)):
            for r in sorted({1, t * t, t * t + 5, 2 * t * t + 1}):
                snf = strassen_basis.random_gaussian_init(t, r, rng, scale=0.5)
                x = rng.standard_normal((bi * t, bk * t))
                w = rng.standard_normal((bk * t, bj * t))
                w_enc = snf_operator.encode_tiles(w, snf.e_w, t)
                x_enc = snf_operator.encode_tiles(x, snf.e_x, t)
                prods = snf_operator._slice_products(x_enc, w_enc)
                cases[f"c{idx}"] = dict(
                    t=t, r=r, x=x, w=w, e_x=snf.e_x, e_w=snf.e_w, d=snf.d, w_enc=w_enc,
                    x_enc=x_enc, prods=prods,
                    decoded=snf_operator.decode_tiles(prods, snf.d, t),
                    batched=snf_operator.stl_batched(x, w_enc, snf),
                    reference=snf_operator.stl_reference(x, w, snf),
                )
                idx += 1
    flat = {}
    for name, c in cases.items():
        for k, v in c.items():
            flat[f"{name}/{k}"] = np.asarray(v)
    np.savez_compressed(OUT / "operator_grid.npz", **flat)

    # 2. Strassen rank-49 factors (exact) and an exactness case
    s49 = strassen_basis.strassen_rank49()
    x = rng.standard_normal((16, 16))
    w = rng.standard_normal((16, 16))
    np.savez_compressed(
        OUT / "strassen49.npz", e_x=s49.e_x, e_w=s49.e_w, d=s49.d, x=x, w=w,
        batched=snf_operator.stl_batched(x, snf_operator.encode_tiles(w, s49.e_w, 4), s49),
        matmul=st.matmul(x, w))

    # 3. random_gaussian_init stream (seeded) and pruned subset
    g = strassen_basis.random_gaussian_init(4, 24, st.make_rng(0), scale=0.5)
    sub = strassen_basis.pruned_subset_init(s49, 24, st.make_rng(7))
    np.savez_compressed(OUT / "fixtures.npz", rg_e_x=g.e_x, rg_e_w=g.e_w, rg_d=g.d,
                        sub_e_x=sub.e_x, sub_e_w=sub.e_w, sub_d=sub.d)

    # 4. layer forward (cached) and backward, two shapes
    lay = {}
    for i, (M, K, N, t, r) in enumerate(((16, 8, 12, 4, 12), (32, 16, 24, 4, 24),
                                         (12, 6, 4, 2, 7))):
        snf = strassen_basis.random_gaussian_init(t, r, rng, scale=0.4)
        w0 = rng.standard_normal((K, N)) / np.sqrt(K)
        layer = toy_network.StlLayer(snf, snf_operator.encode_tiles(w0, snf.e_w, t))
        x = rng.standard_normal((M, K))
        gy = rng.standard_normal((M, N))
        y, cache = toy_network._layer_forward_cached(layer, x)
        g_ex, g_d, g_w, g_x = toy_network._layer_backward(layer, cache, gy)
        for k, v in dict(t=t, r=r, x=x, gy=gy, weights=layer.weights, e_x=snf.e_x, e_w=snf.e_w,
                         d=snf.d, y=y, y_fwd=toy_network.stl_layer_forward(layer, x),
                         u=cache[1], y_enc=cache[2], g_ex=g_ex, g_d=g_d, g_w=g_w,
                         g_x=g_x).items():
            lay[f"l{i}/{k}"] = np.asarray(v)
    np.savez_compressed(OUT / "layer.npz", **lay)

    # 5. fused step (Algorithm 2) two-layer chain
    snf = strassen_basis.random_gaussian_init(4, 20, rng, scale=0.5)
    x = rng.standard_normal((8, 12))
    w1 = rng.standard_normal((12, 8))
    w2 = rng.standard_normal((8, 16))
    enc1 = snf_operator.encode_tiles(w1, snf.e_w, 4)
    enc2 = snf_operator.encode_tiles(w2, snf.e_w, 4)
    h = snf_operator._slice_products(snf_operator.encode_tiles(x, snf.e_x, 4), enc1)
    fused = snf_operator.stl_fused_step(h, enc2, snf)
    np.savez_compressed(OUT / "fused_step.npz", e_x=snf.e_x, e_w=snf.e_w, d=snf.d, x=x,
                        enc1=enc1, enc2=enc2, h=h, fused=fused,
                        decoded=snf_operator.decode_tiles(fused, snf.d, 4),
                        sequential=snf_operator.stl_batched(
                            snf_operator.stl_batched(x, enc1, snf), enc2, snf))

    # 6. cost model golden values (cost_model.py closed forms)
    rows = []
    for n, t, r in ((8192, 4, 32), (8192, 4, 24), (8192, 4, 49), (4096, 2, 16), (1024, 4, 24)):
        s, nv = cost_model.flops_square(n, t, r)
        io, io_n, steps = cost_model.io_square(n, t, r, 2)
        rows.append([n, t, r, s, nv, io, io_n, *steps,
                     cost_model.io_fused_chain(n, t, r, 3, 2),
                     cost_model.flops_general(cost_model.ProblemShape(n, n // 2, n, t, r))])
    np.savez_compressed(OUT / "cost_model.npz", rows=np.array(rows, dtype=np.int64))
    # 7. seeded streams of the remaining fixture helpers (dense_core.py:152-167,
    #    strassen_basis.py:140-142) and instrumented FLOP counts (cost_model.py:150-187)
    kids = st.spawn_rngs(5, 3)
    counts = []
    for (n, t, r) in ((8, 4, 16), (16, 4, 24), (8, 2, 7), (6, 1, 1)):
        shape = cost_model.ProblemShape(n, n, n, t, r)
        counts.append([n, t, r, cost_model.count_reference_flops(shape),
                       cost_model.flops_general(shape)])
    np.savez_compressed(
        OUT / "streams.npz",
        chain=strassen_basis.nested_subset_chain(st.make_rng(3)),
        chain24=strassen_basis.nested_subset_chain(st.make_rng(11), 24),
        gauss=st.gaussian_matrix(st.make_rng(4), 3, 5),
        spawn=np.stack([k.standard_normal(4) for k in kids]),
        unvec=st.unvec_tile(np.arange(16.0), 4),
        counts=np.array(counts, dtype=np.int64))
    print(f"wrote golden fixtures to {OUT}")


if __name__ == "__main__":
    main()
