"""Golden blobs for the reference file formats, written by the REFERENCE.

Run in the build container (where /root/reference is mounted):

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_interop_golden.py

Writes tests/golden/interop/*: an STLM matrix blob and CSV, SNF triple blobs (Strassen rank 7,
exact in fp32, and a seeded Gaussian triple), an STLE encoded tensor, and a two-layer model
checkpoint, each produced by strassen_tile's own writers (dense_core.save_matrix_blob /
save_matrix_csv, snf_operator.save_triple / save_encoded, toy_network.save_model), plus an
.npz with the values they encode.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "interop"


def main() -> None:
    sys.path.insert(0, str(REF))
    from strassen_tile import dense_core, snf_operator, strassen_basis, toy_network

    OUT.mkdir(parents=True, exist_ok=True)
    rng = dense_core.make_rng(7)
    m = rng.standard_normal((3, 5))
    dense_core.save_matrix_blob(OUT / "matrix.stlm", m)
    dense_core.save_matrix_csv(OUT / "matrix.csv", m)
    s7 = strassen_basis.strassen_rank7()
    snf_operator.save_triple(OUT / "strassen7.snf", s7)
    g = strassen_basis.random_gaussian_init(4, 6, rng, scale=0.5)
    snf_operator.save_triple(OUT / "gauss_t4_r6.snf", g)
    enc = snf_operator.encode_tiles(rng.standard_normal((8, 12)), g.e_x, 4)  # (2, 3, 6)
    snf_operator.save_encoded(OUT / "encoded.stle", enc)
    # two layers (t = 2): Strassen-7 with fp32-exact weights, Gaussian r = 5 with float weights
    w1 = np.round(rng.standard_normal((3, 2, 7)) * 8) / 8
    g2 = strassen_basis.random_gaussian_init(2, 5, rng, scale=0.5)
    w2 = rng.standard_normal((2, 4, 5))
    layers = [toy_network.StlLayer(s7, w1), toy_network.StlLayer(g2, w2)]
    toy_network.save_model(OUT / "model.ckpt", layers)
    np.savez(OUT / "values.npz", m=m, s7_e_x=s7.e_x, s7_e_w=s7.e_w, s7_d=s7.d, g_e_x=g.e_x,
             g_e_w=g.e_w, g_d=g.d, enc=enc, w1=w1, w2=w2, g2_e_x=g2.e_x, g2_e_w=g2.e_w,
             g2_d=g2.d)
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
