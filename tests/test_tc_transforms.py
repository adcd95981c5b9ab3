"""The tcgen05 t = 4 transforms (stl_stream_tc.cu) against the CPU oracle: encode and decode of
bf16 data on the shapes they take (tile columns >= 512, a multiple of 64), every plane-count
regime of the UMMA operands (one K-step with a zero-filled 16-plane box, two overlapping
K-steps, P = 32 exactly; 1..4 eight-plane output groups of the encode), partial units, the
dynamic tail schedule (outputs bit-identical across launches), and the decode + g_ex reduction
through the layer backward."""

import numpy as np
import pytest
import torch

import paper_2503_12211_b200 as stl
from oracle import stl_oracle as O

pytestmark = pytest.mark.gpu


def bf(a):
    t = torch.tensor(a, dtype=torch.float32).to(torch.bfloat16)
    return t.cuda(), t.double().numpy()


def rel(got, ref):
    g = got.double().cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got, float)
    return np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30)


# (12, 2304): 576 tiles per row = a full and a 64-tile unit; (16, 4096): two full units per row;
# (4, 8192): one tile row of four units
@pytest.mark.parametrize("rows,cols", [(12, 2304), (16, 4096), (4, 8192)])
@pytest.mark.parametrize("r", [1, 8, 9, 16, 17, 24, 25, 32])
def test_tc_encode_decode(rows, cols, r):
    rng = O.make_rng(rows * 7 + cols + r)
    e_x, _, d = O.random_gaussian_init(4, r, rng, scale=0.5)
    m_dev, m64 = bf(rng.standard_normal((rows, cols)))
    enc = stl.encode_tiles(m_dev, e_x, 4)
    ref_enc = O.encode_tiles(m64, e_x, 4)
    assert rel(enc, ref_enc) <= 5e-3
    enc_dev, enc64 = bf(ref_enc)
    dec = stl.decode_tiles(enc_dev.permute(2, 0, 1).contiguous().permute(1, 2, 0), d, 4)
    assert rel(dec, O.decode_tiles(enc64, d, 4)) <= 5e-3


def test_tc_dynamic_schedule_bitwise():
    """The last third of the units go to whichever CTA asks first: the unit -> SM mapping changes
    from launch to launch, the outputs must not."""
    dev = torch.device("cuda")
    snf = stl.random_gaussian_init(4, 24, stl.make_rng(3), scale=0.5).to(dev)
    g = torch.Generator(device=dev).manual_seed(5)
    x = torch.randn((8192, 4096), device=dev, generator=g).to(torch.bfloat16)
    ref_u = stl.encode_tiles(x, snf.e_x, 4).clone()
    ref_y = stl.decode_tiles(ref_u, snf.d, 4).clone()
    for _ in range(20):
        u = stl.encode_tiles(x, snf.e_x, 4)
        assert torch.equal(u, ref_u)
        assert torch.equal(stl.decode_tiles(u, snf.d, 4), ref_y)


@pytest.mark.parametrize("r", [16, 17, 24, 32])
def test_tc_decode_reduction_backward(r):
    """g_x (decode of g_u) and g_ex (the reduction riding on it) with K / 4 = 1024 tile columns:
    the tcgen05 decode + mma.sync reduction kernel."""
    t, M, K, N = 4, 256, 4096, 2048
    rng = O.make_rng(r + 11)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    x_dev, x64 = bf(rng.standard_normal((M, K)))
    w_dev, w64 = bf(O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t))
    gy_dev, gy64 = bf(rng.standard_normal((M, N)))
    layer = stl.StlLayer(stl.SnfTriple(t, r, e_x, e_w, d), w_dev)
    y, cache = stl._layer_forward_cached(layer, x_dev)
    grads = stl._layer_backward(layer, cache, gy_dev)
    torch.cuda.synchronize()
    y_ref, cache_ref = O.layer_forward_cached(x64, w64, e_x, d, t)
    assert rel(y, y_ref) <= 1e-2
    refs = O.layer_backward(w64, e_x, d, cache_ref, gy64, t)
    for name, g, ref in zip(("g_ex", "g_d", "g_w", "g_x"), grads, refs):
        assert rel(g, ref) <= 1e-2, (name, rel(g, ref))


@pytest.mark.parametrize("r", [8, 16, 24, 32])
def test_tc_remix_chain(r):
    """The fused-chain remix on tcgen05 (block columns 512): a bf16 chain of two fused steps
    against the oracle chain on the same bf16 weights."""
    t, n = 4, 2048
    rng = O.make_rng(200 + r)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    snf = stl.SnfTriple(t, r, e_x, e_w, d)
    x_dev, x64 = bf(rng.standard_normal((n, n)))
    w_dev, w64 = [], []
    for _ in range(3):
        a, b = bf(O.encode_tiles(rng.standard_normal((n, n)) / np.sqrt(n), e_w, t))
        w_dev.append(a)
        w64.append(b)
    h = stl._slice_products(stl.encode_tiles(x_dev, snf.e_x, t), w_dev[0]).to(torch.bfloat16)
    h64 = O.slice_products(O.encode_tiles(x64, e_x, t), w64[0])
    for wd, w6 in zip(w_dev[1:], w64[1:]):
        h = stl.stl_fused_step(h, wd, snf)
        assert h.dtype == torch.bfloat16
        h64 = O.stl_fused_step(h64, w6, e_x, d)
    got = stl.decode_tiles(h, snf.d, t)
    assert rel(got, O.decode_tiles(h64, d, t)) <= 1e-2


def test_tc_strided_and_concurrent():
    """Through the C ABI: a matrix with a padded leading dimension (ld = cols + 64) into and out of
    the tcgen05 encode / decode, and the same encode launched on two streams at once many times
    (the dynamic tail's counter slots must not collide): every result bit-identical."""
    from paper_2503_12211_b200 import _lib

    lib = _lib.load()
    dev = torch.device("cuda")
    rows, cols, ld, r = 64, 4096, 4096 + 64, 24
    rng = O.make_rng(41)
    e_x, _, d = O.random_gaussian_init(4, r, rng, scale=0.5)
    ex = torch.tensor(e_x, dtype=torch.float32, device=dev)
    dd = torch.tensor(d, dtype=torch.float32, device=dev)
    m_dev, m64 = bf(rng.standard_normal((rows, cols)))
    wide = torch.zeros((rows, ld), dtype=torch.bfloat16, device=dev)
    wide[:, :cols] = m_dev
    planes = torch.empty((r, rows // 4, cols // 4), dtype=torch.bfloat16, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.stl_encode(wide.data_ptr(), _lib.STL_BF16, rows, cols, ld, ex.data_ptr(), 4, r,
                              planes.data_ptr(), _lib.STL_BF16, s))
    ref_enc = O.encode_tiles(m64, e_x, 4)
    assert rel(planes.permute(1, 2, 0), ref_enc) <= 5e-3
    out = torch.full((rows, ld), 7.0, dtype=torch.bfloat16, device=dev)
    _lib.check(lib.stl_decode(planes.data_ptr(), _lib.STL_BF16, rows // 4, cols // 4, r,
                              dd.data_ptr(), 4, out.data_ptr(), _lib.STL_BF16, ld, s))
    torch.cuda.synchronize()
    enc64 = planes.permute(1, 2, 0).double().cpu().numpy()
    assert rel(out[:, :cols], O.decode_tiles(enc64, d, 4)) <= 5e-3
    assert torch.all(out[:, cols:] == 7.0)  # the padding columns are never written

    big = torch.randn((4096, 4096), device=dev).to(torch.bfloat16)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = [torch.empty((r, 1024, 1024), dtype=torch.bfloat16, device=dev) for _ in range(2)]
    torch.cuda.synchronize()
    _lib.check(lib.stl_encode(big.data_ptr(), _lib.STL_BF16, 4096, 4096, 4096, ex.data_ptr(), 4, r,
                              outs[0].data_ptr(), _lib.STL_BF16, s))
    torch.cuda.synchronize()
    ref = outs[0].clone()
    for _ in range(50):
        for st, o in zip((s1, s2), outs):
            _lib.check(lib.stl_encode(big.data_ptr(), _lib.STL_BF16, 4096, 4096, 4096, ex.data_ptr(),
                                      4, r, o.data_ptr(), _lib.STL_BF16, st.cuda_stream))
    torch.cuda.synchronize()
    assert torch.equal(outs[0], ref) and torch.equal(outs[1], ref)


@pytest.mark.parametrize("rows,cols", [(8, 2304), (4, 4096)])
@pytest.mark.parametrize("r", [1, 4, 5, 8, 9, 17, 24, 32])
def test_tc_t2_encode_decode(rows, cols, r):
    """t = 2 on tcgen05 (k_encode2_tc / k_decode2_tc): 1152 tile columns = two full units and a
    partial one, every 4-plane output-group count and both K-step regimes of the decode."""
    rng = O.make_rng(rows * 13 + cols + r)
    e_x, _, d = O.random_gaussian_init(2, r, rng, scale=0.5)
    m_dev, m64 = bf(rng.standard_normal((rows, cols)))
    enc = stl.encode_tiles(m_dev, e_x, 2)
    ref_enc = O.encode_tiles(m64, e_x, 2)
    assert rel(enc, ref_enc) <= 5e-3
    enc_dev, enc64 = bf(ref_enc)
    dec = stl.decode_tiles(enc_dev.permute(2, 0, 1).contiguous().permute(1, 2, 0), d, 2)
    assert rel(dec, O.decode_tiles(enc64, d, 2)) <= 5e-3
