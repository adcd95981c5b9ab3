"""The HBM-streaming t = 4 transforms (stl_stream.cu) over their configuration space, against
the CPU oracle: encode / decode of bf16 data with partial units (tile columns not a multiple of
the 512-tile unit), ranks that are not multiples of 8 or 16 (zero-padded plane boxes), every
plane group count (r up to 64), and the fused reductions (g_d, g_ex) through the layer backward
in all three slice-product formats (F24, fp32, bf16 cache)."""

import numpy as np
import pytest
import torch

import paper_2503_12211_b200 as stl
from paper_2503_12211_b200 import _lib
from oracle import stl_oracle as O

pytestmark = pytest.mark.gpu


def bf(a):
    t = torch.tensor(a, dtype=torch.float32).to(torch.bfloat16)
    return t.cuda(), t.double().numpy()


def rel(got, ref):
    g = got.double().cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got, float)
    return np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30)


# (36, 256), (148, 256), (128, 512), (52, 512): narrow matrices, units of 4 / 2 whole tile rows
# with a partial last unit
@pytest.mark.parametrize("rows,cols", [(64, 2304), (36, 256), (8, 4096), (128, 512), (148, 256),
                                       (52, 512)])
@pytest.mark.parametrize("r", [5, 20, 24, 40, 64])
def test_encode_decode_bf16(rows, cols, r):
    """bf16 matrix -> bf16 planes -> bf16 matrix (units: 512 tiles; 2304/4 = 576 = 512 + 64;
    narrow matrices: 256-tile units of several tile rows)."""
    rng = O.make_rng(rows * 31 + cols + r)
    e_x, _, d = O.random_gaussian_init(4, r, rng, scale=0.5)
    m_dev, m64 = bf(rng.standard_normal((rows, cols)))
    enc = stl.encode_tiles(m_dev, e_x, 4)                     # (rows/4, cols/4, r) view
    ref_enc = O.encode_tiles(m64, e_x, 4)
    assert rel(enc, ref_enc) <= 5e-3                            # bf16 output rounding
    enc_dev, enc64 = bf(ref_enc)
    dec = stl.decode_tiles(enc_dev.permute(2, 0, 1).contiguous().permute(1, 2, 0), d, 4)
    assert dec.dtype == torch.bfloat16
    assert rel(dec, O.decode_tiles(enc64, d, 4)) <= 5e-3


@pytest.mark.parametrize("M,K,N,r,fmt", [
    (1024, 512, 512, 24, "bf16"),    # default: bf16 slice products (cache and g_u)
    (1024, 512, 512, 24, "f24"),     # forced F24 slice products (N/4 % 128 == 0)
    (1024, 512, 768, 24, "bf16"),    # N/4 = 192: bf16 products need N/4 % 64 only
    (1024, 2304, 512, 20, "f24"),    # partial 512-tile units in K, r not a multiple of 8
    (1024, 2304, 512, 20, "bf16"),
    (768, 256, 1024, 13, "f24"),     # r = 13: one plane group, zero-padded to 16 in the box
    (768, 256, 1024, 13, "bf16"),
    (1024, 512, 512, 32, "fp32"),    # forced fp32 products, bf16 cache copy
])
def test_layer_fwd_bwd_formats(M, K, N, r, fmt):
    t = 4
    rng = O.make_rng(M + K + N + r)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    x_dev, x64 = bf(rng.standard_normal((M, K)))
    w_dev, w64 = bf(O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t))
    gy_dev, gy64 = bf(rng.standard_normal((M, N)))
    layer = stl.StlLayer(stl.SnfTriple(t, r, e_x, e_w, d), w_dev)
    products = {"bf16": None, "f24": "f24", "fp32": torch.float32}[fmt]
    y, cache = stl._layer_forward_cached(layer, x_dev, products=products)
    grads = stl._layer_backward(layer, cache, gy_dev)
    torch.cuda.synchronize()
    nbytes = cache.y_enc.numel() * cache.y_enc.element_size()
    assert nbytes == {"f24": 3, "bf16": 2, "fp32": 2}[fmt] * r * (M // 4) * (N // 4)
    y_ref, cache_ref = O.layer_forward_cached(x64, w64, e_x, d, t)
    assert rel(y, y_ref) <= 1e-2
    y_enc = stl.unpack_slice_products(cache.y_enc, r, M // 4, N // 4)
    tol_enc = {"f24": 2e-3, "bf16": 5e-3, "fp32": 5e-3}[fmt]  # u is bf16 in all
    assert rel(y_enc, cache_ref[2].transpose(2, 0, 1)) <= tol_enc
    refs = O.layer_backward(w64, e_x, d, cache_ref, gy64, t)
    for name, g, ref in zip(("g_ex", "g_d", "g_w", "g_x"), grads, refs):
        assert rel(g, ref) <= 1e-2, (name, rel(g, ref))


def test_cache_format_is_explicit():
    """The cache's format is an argument, not process state: a format the shape cannot use is
    a ValueError (forward), and a backward told a format the forward could not have written
    fails instead of misreading the bytes (include/stl_b200.h stl_backward_ex)."""
    t, r, M, K, N = 4, 24, 1024, 512, 768  # N/4 = 192: bf16 products yes, F24 no
    rng = O.make_rng(9)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    x_dev, _ = bf(rng.standard_normal((M, K)))
    w_dev, _ = bf(O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t))
    layer = stl.StlLayer(stl.SnfTriple(t, r, e_x, e_w, d), w_dev)
    with pytest.raises(ValueError):
        stl._layer_forward_cached(layer, x_dev, products="f24")
    assert stl.cache_format(M, K, N, t, r, torch.bfloat16) == _lib.STL_BF16
    assert stl.cache_format(M, K, N, t, r, torch.float32) == _lib.STL_F32
    y, cache = stl._layer_forward_cached(layer, x_dev)
    lib = _lib.load()
    dev = x_dev.device
    bi, bk, bj = M // t, K // t, N // t
    g_enc = torch.empty((r, bi, bj), dtype=torch.bfloat16, device=dev)
    g_u = torch.empty((r, bi, bk), dtype=torch.float32, device=dev)
    g_x = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
    snf = layer.snf.on(dev)
    for bad in (_lib.STL_F24, _lib.STL_F32, 7):
        st = lib.stl_backward_ex(
            x_dev.data_ptr(), K, x_dev.data_ptr(), K, layer.w_planes.data_ptr(),
            snf.e_x.data_ptr(), snf.d.data_ptr(), cache.u.data_ptr(), cache.y_enc.data_ptr(), bad,
            M, K, N, t, r, _lib.STL_BF16, None, None, None, g_x.data_ptr(), K, g_enc.data_ptr(),
            g_u.data_ptr(), None, _lib.STL_PROD_AUTO, None, torch.cuda.current_stream().cuda_stream)
        assert st == 2, bad  # STL_ERR_VALUE
    torch.cuda.synchronize()


def test_stage_protocol_under_data_only_probe():
    """Regression for the stage-reuse race (two consumer groups, odd stage counts): with the
    STL_STREAM_NOCOMPUTE probe the consumers only move data, so a group runs far ahead of the
    other; without the producer's per-stage unit tags this faulted within a few hundred
    config-2 steps."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    # the probe switch lives in the probe build of the library only
    env = dict(os.environ, STL_LIB=str(_lib.PROBE_LIB_PATH), STL_STREAM_NOCOMPUTE="1",
               STRESS_STEPS="300")
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "stress_step.py")],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "stress ok" in out.stdout, out.stderr[-2000:]


def test_stage_protocol_bitwise_repeat_with_compute():
    """The same race with the math on: config-2 steps whose reductions run two consumer groups
    over odd stage counts (decode_gu+g_ex: 3 stages, encode_gy+g_d: 7) must reproduce every
    gradient bit for bit across repeated steps (a stale-stage read would change values without
    faulting)."""
    from paper_2503_12211_b200.layer import LayerCache, backward_raw
    from paper_2503_12211_b200.snf_operator import _forward

    T, R, M, K, N = 4, 24, 8192, 4096, 4096
    dev = torch.device("cuda")
    snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
    g = torch.Generator(device=dev).manual_seed(4)
    w = (torch.randn((R, N // T, K // T), device=dev, generator=g) * 0.03).to(torch.bfloat16)
    x = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
    gy = torch.randn((M, N), device=dev, generator=g).to(torch.bfloat16)
    first = None
    for _ in range(40):
        y, u, ye = _forward(x, w, snf, keep_cache=True)
        grads = backward_raw(snf, w, LayerCache(x, u, ye), gy)
        out = [y] + [gr for gr in grads]
        if first is None:
            first = [o.clone() for o in out]
        else:
            for a, b in zip(out, first):
                assert torch.equal(a, b)
    torch.cuda.synchronize()


# ---------------------------------------------------------------- t = 2 (stl_transform2.cu)
@pytest.mark.parametrize("rows,cols", [(64, 2048), (130, 72), (6, 520), (256, 36)])
@pytest.mark.parametrize("r", [3, 16, 24, 32, 49])
def test_encode_decode_t2_bf16(rows, cols, r):
    """t = 2 register-streaming encode / decode (4 tiles per thread; tile columns % 4 == 0) and
    the generic fallback (cols / 2 = 36 / 18: not a multiple of 4), bf16 and fp32 planes."""
    rng = O.make_rng(rows * 7 + cols + r)
    e_x, _, d = O.random_gaussian_init(2, r, rng, scale=0.5)
    m_dev, m64 = bf(rng.standard_normal((rows, cols)))
    enc = stl.encode_tiles(m_dev, e_x, 2)
    ref_enc = O.encode_tiles(m64, e_x, 2)
    assert rel(enc, ref_enc) <= 5e-3
    enc_dev, enc64 = bf(ref_enc)
    dec = stl.decode_tiles(enc_dev.permute(2, 0, 1).contiguous().permute(1, 2, 0), d, 2)
    assert dec.dtype == torch.bfloat16
    assert rel(dec, O.decode_tiles(enc64, d, 2)) <= 5e-3
    enc32 = torch.tensor(ref_enc, dtype=torch.float32, device="cuda")
    dec32 = stl.decode_tiles(enc32.permute(2, 0, 1).contiguous().permute(1, 2, 0), d, 2)
    assert rel(dec32, O.decode_tiles(ref_enc, d, 2)) <= 1e-5


@pytest.mark.parametrize("M,K,N,r", [(1024, 512, 768, 16), (1024, 256, 1024, 24),
                                     (520, 256, 264, 32)])
def test_forward_t2_bf16_products(M, K, N, r):
    """Cache-less bf16 forward at t = 2: bf16 slice products (STL_PROD_AUTO) decoded by the
    t = 2 streaming kernel; within the bf16 bar of the oracle."""
    t = 2
    rng = O.make_rng(M + 3 * K + N + r)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    x_dev, x64 = bf(rng.standard_normal((M, K)))
    w_dev, w64 = bf(O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t))
    fmt = stl.cache_format(M, K, N, t, r, torch.bfloat16, None)
    y = stl.stl_batched(x_dev, w_dev, stl.SnfTriple(t, r, e_x, e_w, d))
    torch.cuda.synchronize()
    assert rel(y, O.stl_batched(x64, w64, e_x, d, t)) <= 1e-2
    assert fmt in (_lib.STL_BF16, _lib.STL_F32)  # the training cache keeps fp32 products at t = 2
