"""Reference file formats: STLM / CSV matrices, SNF triples, STLE encoded
tensors and model checkpoints, against blobs written by the reference itself
(oracle/gen_interop_golden.py -> tests/golden/interop/)."""

from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2503_12211_b200 import interop
from paper_2503_12211_b200.dense_core import ShapeError

G = Path(__file__).resolve().parent / "golden" / "interop"
V = np.load(G / "values.npz")


def _snf64(prefix):
    return SimpleNamespace(t=4 if prefix == "g" else 2, r=V[f"{prefix}_e_x"].shape[0],
                           e_x=V[f"{prefix}_e_x"], e_w=V[f"{prefix}_e_w"], d=V[f"{prefix}_d"])


def test_matrix_blob_and_csv_bytes():
    raw = (G / "matrix.stlm").read_bytes()
    m, end = interop.matrix_from_bytes(raw)
    assert end == len(raw) and np.array_equal(m, V["m"])
    assert interop.matrix_to_bytes(V["m"]) == raw
    assert np.array_equal(interop.load_matrix_csv(G / "matrix.csv"), V["m"])
    assert interop.matrix_to_csv(V["m"]) == (G / "matrix.csv").read_text()


def test_triples():
    s7 = interop.load_triple(G / "strassen7.snf")
    assert (s7.t, s7.r) == (2, 7)
    for k in ("e_x", "e_w", "d"):
        assert np.array_equal(getattr(s7, k).double().numpy(), V[f"s7_{k}"])
    # Strassen factors are fp32-exact: the fp32-held triple writes the same bytes back
    assert interop.triple_to_bytes(s7) == (G / "strassen7.snf").read_bytes()
    g = interop.load_triple(G / "gauss_t4_r6.snf")
    for k in ("e_x", "e_w", "d"):
        np.testing.assert_allclose(getattr(g, k).double().numpy(), V[f"g_{k}"], rtol=1e-7)
    assert interop.triple_to_bytes(_snf64("g")) == (G / "gauss_t4_r6.snf").read_bytes()


def test_encoded_blob():
    raw = (G / "encoded.stle").read_bytes()
    enc, end = interop.encoded_from_bytes(raw)
    assert end == len(raw) and enc.shape == (2, 3, 6) and np.array_equal(enc, V["enc"])
    assert interop.encoded_to_bytes(V["enc"]) == raw


def test_model_checkpoint():
    raw = (G / "model.ckpt").read_bytes()
    layers = interop.model_from_bytes(raw)
    assert len(layers) == 2
    (s1, w1), (s2, w2) = layers
    assert (s1.t, s1.r, s2.t, s2.r) == (2, 7, 2, 5)
    assert np.array_equal(w1, V["w1"]) and np.array_equal(w2, V["w2"])
    s7 = SimpleNamespace(t=2, r=7, e_x=V["s7_e_x"], e_w=V["s7_e_w"], d=V["s7_d"])
    g2 = SimpleNamespace(t=2, r=5, e_x=V["g2_e_x"], e_w=V["g2_e_w"], d=V["g2_d"])
    assert interop.model_to_bytes([(s7, V["w1"]), (g2, V["w2"])]) == raw


@pytest.mark.parametrize("blob,fn", [(b"XXXX" + bytes(20), interop.matrix_from_bytes),
                                     (b"STLM" + bytes(3), interop.matrix_from_bytes),
                                     (b"XXXX" + bytes(28), interop.encoded_from_bytes)])
def test_bad_blobs(blob, fn):
    with pytest.raises(ValueError):
        fn(blob)


def test_version_and_truncation():
    raw = bytearray((G / "matrix.stlm").read_bytes())
    raw[4] = 9
    with pytest.raises(ValueError, match="version"):
        interop.matrix_from_bytes(bytes(raw))
    with pytest.raises(ValueError, match="truncated"):
        interop.matrix_from_bytes((G / "matrix.stlm").read_bytes()[:-8])
    with pytest.raises(ValueError):
        interop.triple_from_bytes(b"no header line")
    with pytest.raises(ShapeError):
        interop.matrix_from_csv("1,2\n3\n")


@pytest.mark.gpu
def test_checkpoint_onto_gpu_layers():
    """A reference checkpoint loads into GPU StlLayers whose forward matches the oracle."""
    import torch

    import paper_2503_12211_b200 as stl
    from oracle import stl_oracle as O

    layers = interop.load_model(G / "model.ckpt")
    x = np.random.default_rng(0).standard_normal((8, layers[0].in_dim))
    h = torch.tensor(x, dtype=torch.float32, device="cuda")
    ref = x
    for layer, (snf, w) in zip(layers, interop.model_from_bytes((G / "model.ckpt").read_bytes())):
        h = stl.stl_layer_forward(layer, h)
        ref = O.stl_batched(ref, w, snf.e_x.double().numpy(), snf.d.double().numpy(), snf.t)
    torch.cuda.synchronize()
    assert O.rel_frobenius(h.double().cpu().numpy(), ref) <= 1e-5
    # and back: the GPU layers serialise to a checkpoint the reader accepts unchanged
    again = interop.model_from_bytes(interop.model_to_bytes(layers))
    assert all(np.allclose(a[1], b.weights.double().cpu().numpy()) for a, b in zip(again, layers))
