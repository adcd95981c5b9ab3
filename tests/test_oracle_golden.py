"""Pin the CPU oracle (oracle/stl_oracle.py) to the reference's own outputs.

The golden vectors in tests/golden/ were produced by running the reference package
(strassen_tile, /root/reference/pkg/src) in the build container via oracle/gen_golden.py.
"""

import numpy as np
import pytest

from oracle import stl_oracle as O
from oracle.golden import golden_cases, load_golden

GRID = golden_cases("operator_grid")


@pytest.mark.parametrize("case", sorted(GRID))
def test_operator_grid(case):
    c = GRID[case]
    t = int(c["t"])
    x_enc = O.encode_tiles(c["x"], c["e_x"], t)
    w_enc = O.encode_tiles(c["w"], c["e_w"], t)
    np.testing.assert_allclose(x_enc, c["x_enc"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(w_enc, c["w_enc"], rtol=0, atol=1e-12)
    prods = O.slice_products(c["x_enc"], c["w_enc"])
    np.testing.assert_allclose(prods, c["prods"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(O.decode_tiles(c["prods"], c["d"], t), c["decoded"], atol=1e-11)
    batched = O.stl_batched(c["x"], c["w_enc"], c["e_x"], c["d"], t)
    scale = max(np.linalg.norm(c["batched"]), 1.0)
    assert np.linalg.norm(batched - c["batched"]) <= 1e-12 * scale
    loop = O.stl_reference_loop(c["x"], c["w"], c["e_x"], c["e_w"], c["d"], t)
    assert np.linalg.norm(loop - c["reference"]) <= 1e-12 * max(np.linalg.norm(c["reference"]), 1.0)
    fast = O.stl_batched_reference_numpy(c["x"], c["w_enc"], c["e_x"], c["d"], t)
    assert np.linalg.norm(fast - c["batched"]) <= 1e-12 * scale


def test_strassen49_factors_and_exactness():
    g = load_golden("strassen49")
    e_x, e_w, d = O.strassen_rank49()
    assert np.array_equal(e_x, g["e_x"]) and np.array_equal(e_w, g["e_w"]) and np.array_equal(d, g["d"])
    w_enc = O.encode_tiles(g["w"], e_w, 4)
    got = O.stl_batched(g["x"], w_enc, e_x, d, 4)
    assert np.abs(got - g["batched"]).max() <= 1e-12
    assert np.abs(got - g["matmul"]).max() <= 1e-9


def test_random_gaussian_stream():
    g = load_golden("fixtures")
    e_x, e_w, d = O.random_gaussian_init(4, 24, O.make_rng(0), scale=0.5)
    assert np.array_equal(e_x, g["rg_e_x"]) and np.array_equal(e_w, g["rg_e_w"])
    assert np.array_equal(d, g["rg_d"])


LAYER = golden_cases("layer")


@pytest.mark.parametrize("case", sorted(LAYER))
def test_layer_forward_backward(case):
    c = LAYER[case]
    t = int(c["t"])
    y, cache = O.layer_forward_cached(c["x"], c["weights"], c["e_x"], c["d"], t)
    np.testing.assert_allclose(y, c["y"], atol=1e-12)
    np.testing.assert_allclose(cache[1], c["u"], atol=1e-12)
    np.testing.assert_allclose(cache[2], c["y_enc"], atol=1e-12)
    for fn in (O.layer_backward, O.layer_backward_einsum):
        g_ex, g_d, g_w, g_x = fn(c["weights"], c["e_x"], c["d"], cache, c["gy"], t)
        for got, key in ((g_ex, "g_ex"), (g_d, "g_d"), (g_w, "g_w"), (g_x, "g_x")):
            np.testing.assert_allclose(got, c[key], rtol=1e-12, atol=1e-12)


def test_fused_step():
    g = load_golden("fused_step")
    fused = O.stl_fused_step(g["h"], g["enc2"], g["e_x"], g["d"])
    np.testing.assert_allclose(fused, g["fused"], atol=1e-11)
    np.testing.assert_allclose(O.decode_tiles(fused, g["d"], 4), g["decoded"], atol=1e-11)
    assert O.rel_frobenius(g["decoded"], g["sequential"]) <= 1e-12


def test_tile_roundtrip_and_errors():
    m = O.make_rng(1).standard_normal((8, 12))
    assert np.array_equal(O.untile_fibers(O.tile_fibers(m, 4), 4), m)
    with pytest.raises(O.ShapeError):
        O.tile_fibers(np.ones((6, 8)), 4)
    with pytest.raises(ValueError):
        O.as_matrix(np.array([[np.nan]]))
