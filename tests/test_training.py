"""Class-0 trainer and fake-encoding machinery against the reference.

Golden runs in tests/golden/training/training.json come from strassen_tile.training itself
(oracle/gen_training_golden.py). The trainer is float64 torch math on the operator's device;
the CPU tests run it on the CPU device, the GPU tests on cuda:0 (and feed the trained triple
through the CUDA operator). The remaining tests restate the reference's own (tests/
test_training.py) identities.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2503_12211_b200 import training as tr
from paper_2503_12211_b200.dense_core import SingularSystemError
from paper_2503_12211_b200.strassen_basis import make_rng, random_gaussian_init, strassen_rank49

GOLDEN = json.loads((Path(__file__).parent / "golden" / "training" / "training.json").read_text())
CPU = torch.device("cpu")


def _np64(snf):
    return [np.asarray(f.detach().cpu().double().numpy() if hasattr(f, "detach") else f)
            for f in (snf.e_x, snf.e_w, snf.d)]


class _T64:
    """float64 numpy triple (the reference's representation) for the machinery's inputs."""

    def __init__(self, t, r, e_x, e_w, d):
        self.t, self.r, self.e_x, self.e_w, self.d = t, r, e_x, e_w, d


def _gauss64(t, r, rng, scale):
    shape = (r, t * t)
    return _T64(t, r, scale * rng.standard_normal(shape), scale * rng.standard_normal(shape),
                scale * rng.standard_normal(shape))


def _check_run(rec, device):
    cfg = tr.Class0Config(**rec["config"])
    if "divergence" in rec:
        with pytest.raises(tr.DivergenceError) as err:
            tr.train_class0(cfg, device=device)
        assert str(err.value) == rec["divergence"]["message"]
        assert [list(p) for p in err.value.curve] == [list(p) for p in rec["divergence"]["curve"]] or \
            np.allclose(np.array(err.value.curve, dtype=float),
                        np.array(rec["divergence"]["curve"], dtype=float), rtol=1e-9, atol=1e-12)
        return
    res, tri = tr.train_class0(cfg, device=device)
    want = rec["result"]
    assert (res.r, res.init, res.seed) == (want["r"], want["init"], want["seed"])
    got_c = np.array(res.loss_curve, dtype=float)
    want_c = np.array(want["loss_curve"], dtype=float)
    assert got_c.shape == want_c.shape
    assert np.array_equal(got_c[:, 0], want_c[:, 0])
    # float64 trajectories: only reduction order differs from numpy/OpenBLAS
    np.testing.assert_allclose(got_c[:, 1], want_c[:, 1], rtol=1e-8, atol=1e-25)
    np.testing.assert_allclose(res.loss_final, want["loss_final"], rtol=1e-8, atol=1e-25)
    for got, ref in zip(tri.factors64, rec["factors"]):
        np.testing.assert_allclose(got.cpu().numpy(), np.array(ref), rtol=1e-7, atol=1e-9)
    # the returned triple is the fp32 copy the GPU operator consumes
    assert tri.e_x.dtype == torch.float32 and tri.r == cfg.r


@pytest.mark.parametrize("idx", range(len(GOLDEN["runs"])))
def test_train_class0_matches_reference(idx):
    _check_run(GOLDEN["runs"][idx], CPU)


def test_losses_match_reference():
    snf = _gauss64(4, 12, make_rng(2), 0.5)
    rng = make_rng(3)
    xs, ws = rng.standard_normal((2000, 4, 4)), rng.standard_normal((2000, 4, 4))
    np.testing.assert_allclose(tr.population_class0_loss(snf, device=CPU),
                               GOLDEN["losses"]["population"], rtol=1e-12)
    np.testing.assert_allclose(tr.class0_loss(snf, list(zip(xs, ws)), device=CPU),
                               GOLDEN["losses"]["monte_carlo"], rtol=1e-12)


def test_gradients_match_reference():
    rng = make_rng(5)
    snf = _gauss64(4, 14, rng, 0.5)
    pair = (rng.standard_normal((4, 4)), rng.standard_normal((4, 4)))
    for got, ref in zip(tr.class0_gradients(snf, pair, device=CPU), GOLDEN["gradients"]):
        np.testing.assert_allclose(got.numpy(), np.array(ref), rtol=1e-11, atol=1e-13)


def test_fake_encoding_matches_reference():
    rng = make_rng(10)
    snf = _gauss64(4, 20, rng, 0.6)
    xs = rng.standard_normal((100, 4, 4))
    w = rng.standard_normal((4, 4))
    f = tr.solution_matrix(snf.e_x, snf.d, xs, device=CPU)
    ref = GOLDEN["fake_encoding"]
    np.testing.assert_allclose(f.numpy(), np.array(ref["solution"]), rtol=1e-8, atol=1e-10)
    reg = tr.per_w_fake_encoding_regression(snf.e_x, snf.d, w, xs, device=CPU)
    np.testing.assert_allclose(reg.numpy(), np.array(ref["regression"]), rtol=1e-8, atol=1e-10)
    fe = f @ torch.from_numpy(w.reshape(-1))
    np.testing.assert_allclose(tr.fake_encoding_loss(snf.e_x, snf.d, fe, w, xs, device=CPU),
                               ref["loss"], rtol=1e-8)


# ------------------------------------------------------------ reference identities
def test_exact_triple_is_zero_and_population_anchors():
    s49 = strassen_rank49()
    rng = make_rng(0)
    pairs = [(rng.standard_normal((4, 4)), rng.standard_normal((4, 4))) for _ in range(20)]
    assert tr.class0_loss(s49, pairs, device=CPU) <= 1e-20
    assert tr.population_class0_loss(s49, device=CPU) <= 1e-20
    z = np.zeros((8, 16))
    zero = _T64(4, 8, z, z, z)
    assert tr.population_class0_loss(zero, device=CPU) == 4.0
    assert tr.class0_loss(zero, [(np.eye(4), np.eye(4))], device=CPU) == 0.25


def test_gradients_zero_at_exact_triple():
    s49 = strassen_rank49()
    rng = make_rng(4)
    pair = (rng.standard_normal((4, 4)), rng.standard_normal((4, 4)))
    for g in tr.class0_gradients(s49, pair, device=CPU):
        assert float(g.abs().max()) <= 1e-12


def test_finite_difference_agreement():
    rng = make_rng(5)
    h = 1e-5
    worst = 0.0
    for _ in range(3):
        snf = _gauss64(4, 14, rng, 0.5)
        pair = (rng.standard_normal((4, 4)), rng.standard_normal((4, 4)))
        grads = tr.class0_gradients(snf, pair, device=CPU)
        for g, arr in zip(grads, (snf.e_x, snf.e_w, snf.d)):
            scale = max(float(g.abs().max()), 1e-12)
            for idx in list(np.ndindex(arr.shape))[::7]:
                old = arr[idx]
                arr[idx] = old + h
                up = tr.class0_loss(snf, [pair], device=CPU)
                arr[idx] = old - h
                dn = tr.class0_loss(snf, [pair], device=CPU)
                arr[idx] = old
                worst = max(worst, abs((up - dn) / (2 * h) - float(g[idx])) / scale)
    assert worst <= 1e-5


def test_zw_vectors_identities():
    rng = make_rng(9)
    e = _gauss64(4, 15, rng, 0.7)
    x = rng.standard_normal((4, 4))
    for i in (0, 7, 15):
        z, zp = tr.build_zw_vectors(x, i, e.e_x, e.d, device=CPU)
        for _ in range(3):
            w = rng.standard_normal((4, 4))
            assert abs(float(z.numpy() @ w.reshape(-1)) - (x @ w).reshape(-1)[i]) <= 1e-12
            fe = rng.standard_normal(15)
            direct = (e.d.T @ ((e.e_x @ x.reshape(-1)) * fe))[i]
            assert abs(float(zp.numpy() @ fe) - direct) <= 1e-12
    z, _ = tr.build_zw_vectors(np.eye(4), 6, e.e_x, e.d, device=CPU)
    assert np.array_equal(z.numpy(), np.eye(16)[6])
    with pytest.raises(IndexError):
        tr.build_zw_vectors(x, 16, e.e_x, e.d, device=CPU)


def test_solution_matrix_singular_and_exact():
    rng = make_rng(13)
    g = _gauss64(4, 20, rng, 1.0)
    with pytest.raises(SingularSystemError) as err:
        tr.solution_matrix(g.e_x, g.d, rng.standard_normal((1, 4, 4)), device=CPU)
    assert err.value.cond is not None
    s49 = strassen_rank49()
    e_x, e_w, d = _np64(s49)
    rng = make_rng(11)
    xs = rng.standard_normal((200, 4, 4))
    f = tr.solution_matrix(e_x, d, xs, device=CPU).numpy()
    for _ in range(3):
        w = rng.standard_normal((4, 4))
        assert tr.fake_encoding_loss(e_x, d, f @ w.reshape(-1), w, xs, device=CPU) <= 1e-8


def test_config_validation():
    with pytest.raises(ValueError):
        tr.Class0Config(r=16, init="mystery").validate()
    with pytest.raises(ValueError):
        tr.Class0Config(r=16, step_size=-1.0).validate()
    with pytest.raises(ValueError):
        tr.train_class0(tr.Class0Config(r=8, t=2), device=CPU)  # strassen subset needs t=4


def test_seed_determinism():
    cfg = tr.Class0Config(r=20, seed=3, steps=100)
    a, _ = tr.train_class0(cfg, device=CPU)
    b, _ = tr.train_class0(tr.Class0Config(r=20, seed=3, steps=100), device=CPU)
    assert a.to_json() == b.to_json() and json.loads(a.to_json())["r"] == 20


# ------------------------------------------------------------ on the GPU
@pytest.mark.gpu
def test_train_class0_on_gpu_matches_reference():
    dev = torch.device("cuda", 0)
    for rec in GOLDEN["runs"]:
        _check_run(rec, dev)


@pytest.mark.gpu
def test_trained_triple_drives_the_operator():
    """A short Class-0 run's triple + fake-encoded init (toy_network.py:239-258) through the CUDA
    layer forward, checked against the same math in float64."""
    from paper_2503_12211_b200 import stl_layer_forward

    dev = torch.device("cuda", 0)
    base = tr.class0_base_triple(r=24, seed=0, encoder_steps=200, device=dev)
    rng = make_rng(1)
    layers = tr.init_stl_layers((64, 128, 32), base, rng, device=dev)
    x = torch.from_numpy(rng.standard_normal((256, 64))).to(dev, torch.float32)
    h = x
    for layer in layers:
        h = stl_layer_forward(layer, h)
    # float64 restatement: per-tile encode, slice products, decode (snf_operator.py:156-172)
    ref = x.double()
    for layer in layers:
        t = layer.snf.t
        ex, d = layer.snf.e_x.double(), layer.snf.d.double()
        w = layer.weights.double()  # (bk, bj, r)
        m, k = ref.shape
        fib = ref.reshape(m // t, t, k // t, t).transpose(1, 2).reshape(m // t, k // t, t * t)
        enc = fib @ ex.T
        prod = torch.einsum("ikp,kjp->ijp", enc, w)
        out = prod @ d
        ref = out.reshape(m // t, -1, t, t).transpose(1, 2).reshape(m, -1)
    err = float((h.double() - ref).norm() / ref.norm())
    assert err <= 1e-5, err
