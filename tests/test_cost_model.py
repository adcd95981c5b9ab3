"""The package's cost model and fixture streams against the reference.

Mirrors /root/reference/pkg/tests/test_cost_model.py (closed forms, report invariants, speedup
table) on this package's ``cost_model`` and pins it to tests/golden/cost_model.npz; pins the
package's seeded fixture helpers (random_gaussian_init, pruned_subset_init, nested_subset_chain,
gaussian_matrix, spawn_rngs, unvec_tile) to streams the reference produced
(tests/golden/fixtures.npz, streams.npz; oracle/gen_golden.py). ``count_reference_flops`` runs
the GPU pipeline, so its tests are ``-m gpu``.
"""

import numpy as np
import pytest

import paper_2503_12211_b200 as stl
from oracle.golden import load_golden
from paper_2503_12211_b200.cost_model import (
    CostReport,
    ProblemShape,
    cost_report,
    count_reference_flops,
    flops_general,
    flops_square,
    io_fused_chain,
    io_square,
    speedup_table,
)


def test_golden_closed_forms():
    for n, t, r, s, nv, io, io_n, s1, s2, s3, chain, gen in load_golden("cost_model")["rows"]:
        n, t, r = int(n), int(t), int(r)
        assert flops_square(n, t, r) == (s, nv)
        assert io_square(n, t, r, 2) == (io, io_n, (s1, s2, s3))
        assert io_fused_chain(n, t, r, 3, 2) == chain
        assert flops_general(ProblemShape(n, n // 2, n, t, r)) == gen


@pytest.mark.parametrize("t,r", [(1, 1), (2, 3), (4, 20)])
def test_single_tile_closed_form(t, r):
    assert flops_general(ProblemShape(t, t, t, t, r)) == 6 * t * t * r + 2 * r


def test_general_vs_square_and_linearity():
    n, t, r = 8192, 4, 32
    assert flops_general(ProblemShape(n, n, n, t, r)) - flops_square(n, t, r)[0] == 2 * n * n * r
    base = flops_general(ProblemShape(64, 64, 64, 4, 16))
    assert flops_general(ProblemShape(64, 64, 64, 4, 32)) == 2 * base


def test_invalid_shape_rejected():
    with pytest.raises(stl.ShapeError):
        ProblemShape(10, 8, 8, 4, 16)
    with pytest.raises(stl.ShapeError):
        ProblemShape(8, 8, 8, 4, 0)
    with pytest.raises(stl.ShapeError):
        io_fused_chain(8, 4, 4, 0)


def test_headline_numbers():
    stl_f, naive = flops_square(8192, 4, 32)
    assert (stl_f, naive) == (558_345_748_480, 1_099_511_627_776)
    io_stl, io_naive, steps = io_square(8192, 4, 32, 2)
    assert io_stl == 12 * 134_217_728 and io_naive == 3 * 134_217_728 and sum(steps) == io_stl
    assert io_square(256, 4, 16, 2)[0] == 7 * (2 * 256 * 256)


def test_speedup_table_and_reports():
    table = speedup_table([16384], [16, 24, 32, 40, 48], 4)
    ratios = [rep.speedup_flops for rep in table]
    assert all(a > b for a, b in zip(ratios, ratios[1:]))
    rows = speedup_table([8, 16], [1, 2], 2, bytes_per_scalar=4)
    assert [(rep.n, rep.r) for rep in rows] == [(8, 1), (8, 2), (16, 1), (16, 2)]
    assert all(isinstance(rep, CostReport) for rep in rows)
    for n, t, r in ((8, 4, 20), (64, 2, 3), (4096, 4, 49)):
        rep = cost_report(n, t, r)
        assert sum(rep.flop_steps) == rep.flops_stl and sum(rep.io_steps) == rep.io_stl_bytes
    rep = cost_report(100 * 64, 4, 49)
    assert abs(rep.speedup_flops - 64 / 49) <= 0.1 * 64 / 49


def test_package_fixture_streams_match_reference():
    """The package's own seeded helpers reproduce the reference's streams (the bench, the T2T
    model and the training path draw from them)."""
    f = load_golden("fixtures")
    g = stl.random_gaussian_init(4, 24, stl.make_rng(0), scale=0.5)
    for name in ("e_x", "e_w", "d"):
        want = np.float32(f[f"rg_{name}"])  # SnfTriple holds fp32 factors
        assert np.array_equal(getattr(g, name).cpu().numpy(), want)
    sub = stl.pruned_subset_init(stl.strassen_rank49(), 24, stl.make_rng(7))
    for name in ("e_x", "e_w", "d"):
        assert np.array_equal(getattr(sub, name).cpu().numpy(), np.float32(f[f"sub_{name}"]))
    s = load_golden("streams")
    assert np.array_equal(stl.nested_subset_chain(stl.make_rng(3)), s["chain"])
    assert np.array_equal(stl.nested_subset_chain(stl.make_rng(11), 24), s["chain24"])
    assert np.array_equal(stl.gaussian_matrix(stl.make_rng(4), 3, 5), s["gauss"])
    kids = stl.spawn_rngs(5, 3)
    assert np.array_equal(np.stack([k.standard_normal(4) for k in kids]), s["spawn"])
    with pytest.raises(stl.ShapeError):
        stl.gaussian_matrix(stl.make_rng(0), 0, 3)


@pytest.mark.gpu
def test_unvec_tile_roundtrip():
    import torch

    s = load_golden("streams")
    tile = stl.unvec_tile(np.arange(16.0), 4)
    assert np.array_equal(tile.cpu().numpy(), s["unvec"])
    m = torch.randn(8, 12, device="cuda")
    assert torch.equal(stl.unvec_tile(stl.vec_tile(m, 1, 2, 4), 4), m[4:8, 8:12])
    with pytest.raises(stl.ShapeError):
        stl.unvec_tile(np.arange(15.0), 4)


@pytest.mark.gpu
def test_count_reference_flops_matches_reference_counts():
    """Instrumented count through the GPU pipeline == the reference's count == flops_general."""
    for n, t, r, counted, general in load_golden("streams")["counts"]:
        shape = ProblemShape(int(n), int(n), int(n), int(t), int(r))
        assert count_reference_flops(shape) == counted == flops_general(shape) == general
    n, t, r = 16, 4, 16
    assert count_reference_flops(ProblemShape(n, n, n, t, r)) == flops_square(n, t, r)[0] + 2 * n * n * r
