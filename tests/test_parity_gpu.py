"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle and the
reference's golden vectors.

Tolerances (BASELINE.json north_star): fp32 within 1e-5 relative Frobenius error, bf16 within
1e-2. bf16 cases round every input to bf16 once and feed the SAME rounded values (upcast to
f64) to the oracle, so the measured error is the kernels' arithmetic, not input quantisation.
"""

import numpy as np
import pytest
import torch

import paper_2503_12211_b200 as stl
from paper_2503_12211_b200 import _lib
from oracle import stl_oracle as O
from oracle.golden import golden_cases, load_golden

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 1e-2
DEV = "cuda"


def f64(t):
    return t.detach().float().cpu().double().numpy() if isinstance(t, torch.Tensor) else np.asarray(t, dtype=np.float64)


def bf16_round(a):
    """Round a numpy array to bf16 and return (torch bf16 cuda tensor, f64 numpy of the same)."""
    t = torch.as_tensor(np.asarray(a), dtype=torch.float32).to(torch.bfloat16)
    return t.to(DEV), t.double().numpy()


def rel(got, ref):
    return O.rel_frobenius(f64(got), f64(ref))


@pytest.fixture(autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    _lib.load()  # fail loudly if the native library is missing
    yield
    torch.cuda.synchronize()


# ----------------------------------------------------------------- golden vectors (fp32)
GRID = golden_cases("operator_grid")


@pytest.mark.parametrize("case", sorted(GRID))
def test_golden_grid_fp32(case):
    c = GRID[case]
    t, r = int(c["t"]), int(c["r"])
    snf = stl.SnfTriple(t, r, c["e_x"], c["e_w"], c["d"])
    x = torch.tensor(c["x"], dtype=torch.float32, device=DEV)
    w = torch.tensor(c["w"], dtype=torch.float32, device=DEV)
    x_enc = stl.encode_tiles(x, snf.e_x, t)
    assert rel(x_enc, c["x_enc"]) <= FP32_TOL
    w_enc = stl.encode_tiles(w, snf.e_w, t)
    assert rel(w_enc, c["w_enc"]) <= FP32_TOL
    prods = stl._slice_products(x_enc, w_enc)
    assert rel(prods, c["prods"]) <= FP32_TOL
    assert rel(stl.decode_tiles(torch.tensor(c["prods"], dtype=torch.float32), snf.d, t),
               c["decoded"]) <= FP32_TOL
    assert rel(stl.stl_batched(x, torch.tensor(c["w_enc"], dtype=torch.float32), snf),
               c["batched"]) <= FP32_TOL
    assert rel(stl.stl_reference(x, w, snf), c["reference"]) <= FP32_TOL


LAYER = golden_cases("layer")


@pytest.mark.parametrize("case", sorted(LAYER))
def test_golden_layer_fp32(case):
    c = LAYER[case]
    t, r = int(c["t"]), int(c["r"])
    layer = stl.StlLayer(stl.SnfTriple(t, r, c["e_x"], c["e_w"], c["d"]),
                         torch.tensor(c["weights"], dtype=torch.float32))
    assert rel(stl.stl_layer_forward(layer, c["x"]), c["y_fwd"]) <= FP32_TOL
    y, cache = stl._layer_forward_cached(layer, c["x"])
    assert rel(y, c["y"]) <= FP32_TOL
    assert rel(cache.u.permute(1, 2, 0), c["u"]) <= FP32_TOL
    assert rel(cache.y_enc.permute(1, 2, 0), c["y_enc"]) <= FP32_TOL
    g_ex, g_d, g_w, g_x = stl._layer_backward(layer, cache, c["gy"])
    for got, key in ((g_ex, "g_ex"), (g_d, "g_d"), (g_w, "g_w"), (g_x, "g_x")):
        assert rel(got, c[key]) <= FP32_TOL, key


def test_golden_fused_step_fp32():
    g = load_golden("fused_step")
    snf = stl.SnfTriple(4, 20, g["e_x"], g["e_w"], g["d"])
    fused = stl.stl_fused_step(torch.tensor(g["h"], dtype=torch.float32),
                               torch.tensor(g["enc2"], dtype=torch.float32), snf)
    assert rel(fused, g["fused"]) <= FP32_TOL
    assert rel(stl.decode_tiles(fused, snf.d, 4), g["decoded"]) <= FP32_TOL


def test_golden_strassen49_exact():
    g = load_golden("strassen49")
    s49 = stl.strassen_rank49()
    for f in ("e_x", "e_w", "d"):
        assert np.array_equal(f64(getattr(s49, f)), g[f])
    x = torch.tensor(g["x"], dtype=torch.float32, device=DEV)
    w = torch.tensor(g["w"], dtype=torch.float32, device=DEV)
    got = stl.stl_batched(x, stl.encode_tiles(w, s49.e_w, 4), s49)
    assert rel(got, g["batched"]) <= FP32_TOL
    assert rel(got, g["matmul"]) <= FP32_TOL


# ----------------------------------------------------------------- config 1 (fp32, 1024^3)
def test_config1_fp32_1024():
    """t=4, r=24, X 1024x1024 . W 1024x1024 fp32, random encoders, seed 0 (BASELINE configs[0])."""
    rng = O.make_rng(0)
    x = rng.standard_normal((1024, 1024))
    w0 = rng.standard_normal((1024, 1024)) / np.sqrt(1024)
    e_x, e_w, d = O.random_gaussian_init(4, 24, rng, scale=0.5)
    w_enc = O.encode_tiles(w0, e_w, 4)
    ref = O.stl_batched(x, w_enc, e_x, d, 4)
    snf = stl.SnfTriple(4, 24, e_x, e_w, d)
    got = stl.stl_batched(torch.tensor(x, dtype=torch.float32, device=DEV),
                          torch.tensor(w_enc, dtype=torch.float32, device=DEV), snf)
    assert got.dtype == torch.float32
    assert rel(got, ref) <= FP32_TOL


# ----------------------------------------------------------------- tcgen05 slice GEMM
def _gemm(a, al, b, bl, M, N, K, r, out_dtype=torch.float32):
    c = torch.empty((r, M, N), dtype=out_dtype, device=DEV)
    _lib.check(_lib.load().stl_slice_gemm(
        a.data_ptr(), al, b.data_ptr(), bl, c.data_ptr(),
        _lib.STL_BF16 if out_dtype == torch.bfloat16 else _lib.STL_F32,
        _lib.STL_BF16 if a.dtype == torch.bfloat16 else _lib.STL_F32, r, M, N, K,
        torch.cuda.current_stream().cuda_stream))
    return c


@pytest.mark.parametrize("al", [0, 1])
@pytest.mark.parametrize("bl", [0, 1])
@pytest.mark.parametrize("shape", [(3, 128, 256, 64), (2, 200, 136, 72), (5, 384, 520, 1000),
                                   (1, 8, 8, 8), (24, 256, 128, 512), (2, 1032, 264, 136)])
def test_slice_gemm_tc_layouts(al, bl, shape):
    """bf16 tcgen05 kernel, every operand-major combination, ragged M/N/K tails."""
    r, M, N, K = shape
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K + al * 2 + bl)
    A = torch.randn((r, M, K), generator=g).to(torch.bfloat16)
    B = torch.randn((r, K, N), generator=g).to(torch.bfloat16)
    ref = torch.bmm(A.double(), B.double())
    a_dev = (A if al == 0 else A.transpose(1, 2)).contiguous().to(DEV)
    b_dev = (B.transpose(1, 2) if bl == 0 else B).contiguous().to(DEV)
    c = _gemm(a_dev, al, b_dev, bl, M, N, K, r)
    err = (c.cpu().double() - ref).norm() / ref.norm()
    assert err <= 1e-5, float(err)
    cb = _gemm(a_dev, al, b_dev, bl, M, N, K, r, out_dtype=torch.bfloat16)
    errb = (cb.cpu().double() - ref).norm() / ref.norm()
    assert errb <= 5e-3, float(errb)


@pytest.mark.parametrize("al,bl", [(0, 0), (1, 1), (0, 1)])
@pytest.mark.parametrize("shape", [(3, 256, 128, 64), (2, 520, 272, 136), (24, 512, 256, 512)])
def test_slice_gemm_f24_output(al, bl, shape):
    """F24 slice products (CTA-pair epilogue): bit-exact RNE-24 of the fp32 products of the
    same kernel, and ~2^-17 relative to the f64 product."""
    r, M, N, K = shape
    g = torch.Generator(device="cpu").manual_seed(M + N + K + 5 * al + bl)
    A = torch.randn((r, M, K), generator=g).to(torch.bfloat16)
    B = torch.randn((r, K, N), generator=g).to(torch.bfloat16)
    a_dev = (A if al == 0 else A.transpose(1, 2)).contiguous().to(DEV)
    b_dev = (B.transpose(1, 2) if bl == 0 else B).contiguous().to(DEV)
    c32 = _gemm(a_dev, al, b_dev, bl, M, N, K, r)
    c24 = torch.empty((3 * r * M * N,), dtype=torch.uint8, device=DEV)
    _lib.check(_lib.load().stl_slice_gemm(a_dev.data_ptr(), al, b_dev.data_ptr(), bl,
                                          c24.data_ptr(), _lib.STL_F24, _lib.STL_BF16, r, M, N, K,
                                          torch.cuda.current_stream().cuda_stream))
    got = stl.unpack_slice_products(c24, r, M, N)
    u = c32.view(torch.int32)
    rne = ((u + 0x7F + ((u >> 8) & 1)) & ~0xFF).view(torch.float32)
    assert torch.equal(got, rne)
    ref = torch.bmm(A.double(), B.double())
    assert (got.cpu().double() - ref).norm() / ref.norm() <= 2e-5


@pytest.mark.parametrize("shape", [(3, 37, 29, 13), (2, 64, 64, 64), (24, 256, 256, 256)])
def test_slice_gemm_simt_fp32(shape):
    r, M, N, K = shape
    g = torch.Generator(device="cpu").manual_seed(11)
    A = torch.randn((r, M, K), generator=g)
    B = torch.randn((r, K, N), generator=g)
    ref = torch.bmm(A.double(), B.double())
    for al, bl in ((0, 0), (0, 1), (1, 1), (1, 0)):
        a_dev = (A if al == 0 else A.transpose(1, 2)).contiguous().to(DEV)
        b_dev = (B.transpose(1, 2) if bl == 0 else B).contiguous().to(DEV)
        c = _gemm(a_dev, al, b_dev, bl, M, N, K, r)
        assert (c.cpu().double() - ref).norm() / ref.norm() <= 1e-6


# ----------------------------------------------------------------- bf16 operator parity
def _bf16_problem(M, K, N, t, r, seed, strassen=False):
    rng = O.make_rng(seed)
    if strassen:
        e_x, e_w, d = O.strassen_rank49()
    else:
        e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    x_dev, x64 = bf16_round(rng.standard_normal((M, K)))
    w0 = rng.standard_normal((K, N)) / np.sqrt(K)
    w_dev_enc, w_enc64 = bf16_round(O.encode_tiles(w0, e_w, t))
    return (e_x, e_w, d), x_dev, x64, w_dev_enc, w_enc64


@pytest.mark.parametrize("M,K,N,t,r,strassen", [
    (1024, 1024, 1024, 4, 24, False),
    (2048, 1024, 512, 4, 16, False),
    (1024, 1024, 1024, 4, 49, True),
    (512, 512, 512, 2, 24, False),
    (768, 256, 1280, 4, 32, False),
])
def test_stl_batched_bf16(M, K, N, t, r, strassen):
    (e_x, e_w, d), x_dev, x64, w_dev, w64 = _bf16_problem(M, K, N, t, r, 3, strassen)
    ref = O.stl_batched(x64, w64, e_x, d, t)
    snf = stl.SnfTriple(t, r, e_x, e_w, d)
    got = stl.stl_batched(x_dev, w_dev, snf)
    assert got.dtype == torch.bfloat16
    err = rel(got, ref)
    assert err <= BF16_TOL, err


@pytest.mark.parametrize("M,K,N,r,init", [
    (2048, 256, 2048, 24, "gaussian"),
    (4096, 512, 2048, 16, "gaussian"),
    (3328, 256, 2560, 32, "gaussian"),   # ragged last 256-row block
    (2048, 512, 2048, 24, "subset"),     # the paper's training init: Strassen-49 row subset
])
def test_forward_backward_bf16_whole_output(M, K, N, r, init):
    """Default bf16 path (bf16 slice products) against the f64 oracle over the whole output
    and in two row slabs, cache-less and with the training cache whose slice products the
    backward then reads; the Strassen-subset r = 24 encoders are the paper's training init."""
    t = 4
    rng = O.make_rng(M + K + r)
    if init == "subset":
        sub = stl.pruned_subset_init(stl.strassen_rank49(), r, stl.make_rng(7))
        e_x, e_w, d = (getattr(sub, n).double().numpy() for n in ("e_x", "e_w", "d"))
    else:
        e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    x_dev, x64 = bf16_round(rng.standard_normal((M, K)))
    w_dev, w64 = bf16_round(O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t))
    snf = stl.SnfTriple(t, r, e_x, e_w, d)
    ref = O.stl_batched(x64, w64, e_x, d, t)
    got = stl.stl_batched(x_dev, w_dev, snf)
    assert rel(got, ref) <= BF16_TOL
    # bands agree separately (a wrong band would hide in the whole-matrix norm)
    half = (M // 4 // 256 // 2) * 256 * 4
    for rows in (slice(0, half), slice(half, M)):
        assert rel(got[rows], ref[rows]) <= BF16_TOL
    layer = stl.StlLayer(snf, w_dev)
    y, cache = stl._layer_forward_cached(layer, x_dev)
    assert torch.equal(y, got)
    y_ref, cache_ref = O.layer_forward_cached(x64, w64, e_x, d, t)
    prods = stl.unpack_slice_products(cache.y_enc, r, M // t, N // t)
    assert rel(prods.permute(1, 2, 0), cache_ref[2]) <= BF16_TOL
    gy_dev, gy64 = bf16_round(rng.standard_normal((M, N)))
    grads = stl._layer_backward(layer, cache, gy_dev)
    refs = O.layer_backward(w64, e_x, d, cache_ref, gy64, t)
    for g_, r_, name in zip(grads, refs, ("g_ex", "g_d", "g_w", "g_x")):
        assert rel(g_, r_) <= BF16_TOL, name


def test_encode_decode_bf16_and_fp32():
    rng = O.make_rng(5)
    for t in (1, 2, 4, 8):
        r = min(2 * t * t + 1, 64)
        enc = rng.standard_normal((r, t * t)) * 0.5
        m = rng.standard_normal((64 * t, 48 * t))
        ref = O.encode_tiles(m, enc, t)
        got = stl.encode_tiles(torch.tensor(m, dtype=torch.float32, device=DEV), enc, t)
        assert rel(got, ref) <= 1e-6
        mb, m64 = bf16_round(m)
        gotb = stl.encode_tiles(mb, enc, t)
        assert gotb.dtype == torch.bfloat16
        assert rel(gotb, O.encode_tiles(m64, enc, t)) <= 5e-3
        planes = rng.standard_normal((64, 48, r))
        dref = O.decode_tiles(planes, enc, t)
        assert rel(stl.decode_tiles(torch.tensor(planes, dtype=torch.float32), enc, t), dref) <= 1e-6


# ----------------------------------------------------------------- layer backward (bf16)
@pytest.mark.parametrize("M,K,N,r", [(1024, 512, 768, 24), (2048, 1024, 1024, 24), (512, 256, 256, 49),
                                     # narrow layers, long token axis: g_w runs split-K
                                     # (1-CTA tiles, S = 4; CTA-pair tiles, S = 2)
                                     (16384, 256, 256, 24), (12800, 256, 768, 24)])
def test_layer_backward_bf16(M, K, N, r):
    t = 4
    rng = O.make_rng(M + r)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    x_dev, x64 = bf16_round(rng.standard_normal((M, K)))
    w_dev, w64 = bf16_round(O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t))
    gy_dev, gy64 = bf16_round(rng.standard_normal((M, N)))
    layer = stl.StlLayer(stl.SnfTriple(t, r, e_x, e_w, d), w_dev)
    y, cache = stl._layer_forward_cached(layer, x_dev)
    y_ref, cache_ref = O.layer_forward_cached(x64, w64, e_x, d, t)
    assert rel(y, y_ref) <= BF16_TOL
    grads = stl._layer_backward(layer, cache, gy_dev)
    refs = O.layer_backward(w64, e_x, d, cache_ref, gy64, t)
    for got, ref, name in zip(grads, refs, ("g_ex", "g_d", "g_w", "g_x")):
        err = rel(got, ref)
        assert err <= BF16_TOL, (name, err)


def test_layer_backward_fp32_moderate():
    t, r, M, K, N = 4, 24, 256, 128, 192
    rng = O.make_rng(77)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    x = rng.standard_normal((M, K))
    w = O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t)
    gy = rng.standard_normal((M, N))
    layer = stl.StlLayer(stl.SnfTriple(t, r, e_x, e_w, d), torch.tensor(w, dtype=torch.float32))
    y, cache = stl._layer_forward_cached(layer, torch.tensor(x, dtype=torch.float32, device=DEV))
    y_ref, cache_ref = O.layer_forward_cached(x, w, e_x, d, t)
    assert rel(y, y_ref) <= FP32_TOL
    for got, ref in zip(stl._layer_backward(layer, cache, gy),
                        O.layer_backward(w, e_x, d, cache_ref, gy, t)):
        assert rel(got, ref) <= FP32_TOL


def test_autograd_module_matches_layer_backward():
    t, r, M, K, N = 4, 24, 512, 256, 512
    rng = O.make_rng(9)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    w = O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t)
    snf = stl.SnfTriple(t, r, e_x, e_w, d)
    layer = stl.StlLayer(snf, torch.tensor(w, dtype=torch.bfloat16))
    mod = stl.StlLinear.from_layer(layer)
    x = torch.randn((M, K), device=DEV).to(torch.bfloat16).requires_grad_(True)
    gy = torch.randn((M, N), device=DEV).to(torch.bfloat16)
    y = mod(x)
    y.backward(gy)
    _, cache = stl._layer_forward_cached(layer, x.detach())
    g_ex, g_d, g_w, g_x = stl._layer_backward(layer, cache, gy)
    assert rel(x.grad, g_x) <= 1e-6
    assert rel(mod.e_x.grad, g_ex) <= 1e-6
    assert rel(mod.d.grad, g_d) <= 1e-6
    assert rel(mod.w_planes.grad.float().permute(2, 1, 0), g_w) <= 1e-2


# ----------------------------------------------------------------- fused step (bf16)
def test_fused_step_bf16():
    t, r = 4, 24
    rng = O.make_rng(21)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    h = rng.standard_normal((256, 128, r))
    w_dev, w64 = bf16_round(O.encode_tiles(rng.standard_normal((512, 384)) / 20, e_w, t))
    ref = O.stl_fused_step(h, w64, e_x, d)
    got = stl.stl_fused_step(torch.tensor(h, dtype=torch.float32), w_dev,
                             stl.SnfTriple(t, r, e_x, e_w, d))
    assert rel(got, ref) <= BF16_TOL


# ----------------------------------------------------------------- full-size properties
def _triple(init, t, r, rng):
    """Random N(0, 0.25) encoders, or the paper's training init: a Strassen-49 row subset."""
    if init == "subset":
        sub = stl.pruned_subset_init(stl.strassen_rank49(), r, rng)
        return tuple(np.asarray(getattr(sub, f).cpu() if hasattr(getattr(sub, f), "cpu")
                                else getattr(sub, f), dtype=np.float64) for f in ("e_x", "e_w", "d"))
    return O.random_gaussian_init(t, r, rng, scale=0.5)


@pytest.mark.parametrize("init", ["gaussian", "subset"])
@pytest.mark.parametrize("M,K,N", [(8192, 4096, 4096), (8192, 8192, 8192)])
def test_full_size_row_slab_and_linearity_bf16(init, M, K, N):
    """BASELINE configs[1] (M=8192, K=N=4096) and north-star (8192^3) shapes, t=4, r=24, through
    the default bf16-product path: rows of Y depend only on the same rows of X, so 64-row slabs
    are checked against the oracle; linearity in x is checked over the whole output."""
    t, r = 4, 24
    rng = O.make_rng(0)
    e_x, e_w, d = _triple(init, t, r, rng)
    w_dev, w64 = bf16_round(O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t))
    snf = stl.SnfTriple(t, r, e_x, e_w, d)
    g = torch.Generator(device=DEV).manual_seed(1)
    x1 = torch.randn((M, K), device=DEV, generator=g).to(torch.bfloat16)
    x2 = torch.randn((M, K), device=DEV, generator=g).to(torch.bfloat16)
    y1 = stl.stl_batched(x1, w_dev, snf)
    for lo in (0, 4096, M - 64):
        slab = x1[lo:lo + 64].float().cpu().double().numpy()
        assert rel(y1[lo:lo + 64], O.stl_batched(slab, w64, e_x, d, t)) <= BF16_TOL
    y2 = stl.stl_batched(x2, w_dev, snf)
    ys = stl.stl_batched((x1.float() + x2.float()).to(torch.bfloat16), w_dev, snf)
    assert rel(ys.float(), y1.float() + y2.float()) <= BF16_TOL


def test_full_size_strassen49_equals_matmul_bf16():
    """An exact triple makes STL a dense matmul: checks the whole 8192x8192x8192 output."""
    M = K = N = 8192
    s49 = stl.strassen_rank49()
    g = torch.Generator(device=DEV).manual_seed(2)
    x = torch.randn((M, K), device=DEV, generator=g).to(torch.bfloat16)
    w = (torch.randn((K, N), device=DEV, generator=g) / 90.0).to(torch.bfloat16)
    w_enc = stl.encode_tiles(w.float(), s49.on(x.device).e_w, 4).to(torch.bfloat16)
    got = stl.stl_batched(x, w_enc, s49)
    ref = x.float() @ w.float()
    assert rel(got.float(), ref) <= BF16_TOL


@pytest.mark.parametrize("init", ["gaussian", "subset"])
def test_full_size_backward_properties_bf16(init):
    """BASELINE configs[1] shape, forward + backward: g_x rows depend only on the same rows of
    gY (64-row slabs against the oracle), and g_w, g_d, g_ex are sums over token rows, so the
    backward of the two halves of the batch must add up to the backward of the whole."""
    t, r, M, K, N = 4, 24, 8192, 4096, 4096
    rng = O.make_rng(5)
    e_x, e_w, d = _triple(init, t, r, rng)
    w_dev, w64 = bf16_round(O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t))
    layer = stl.StlLayer(stl.SnfTriple(t, r, e_x, e_w, d), w_dev)
    g = torch.Generator(device=DEV).manual_seed(6)
    x = torch.randn((M, K), device=DEV, generator=g).to(torch.bfloat16)
    gy = torch.randn((M, N), device=DEV, generator=g).to(torch.bfloat16)

    def fwd_bwd(rows):
        _, cache = stl._layer_forward_cached(layer, x[rows])
        return [gr.float() for gr in stl._layer_backward(layer, cache, gy[rows])]

    g_ex, g_d, g_w, g_x = fwd_bwd(slice(0, M))
    for lo in (0, M - 64):
        rows = slice(lo, lo + 64)
        x64 = x[rows].double().cpu().numpy()
        gy64 = gy[rows].double().cpu().numpy()
        _, cache64 = O.layer_forward_cached(x64, w64, e_x, d, t)
        ref_gx = O.layer_backward(w64, e_x, d, cache64, gy64, t)[3]
        assert rel(g_x[rows], ref_gx) <= BF16_TOL
    halves = [fwd_bwd(slice(0, M // 2)), fwd_bwd(slice(M // 2, M))]
    for i, (name, full) in enumerate((("g_ex", g_ex), ("g_d", g_d), ("g_w", g_w))):
        summed = halves[0][i] + halves[1][i]
        assert rel(summed, full) <= 1e-4, (name, rel(summed, full))
    assert torch.equal(torch.cat([halves[0][3], halves[1][3]]), g_x)


def test_full_size_strassen49_backward_equals_matmul_bf16():
    """With an exact triple the layer is Y = X W, so its input gradient is gY W^T: checked over
    the whole output at M = 8192, K = N = 4096 (fp32 slice products at r = 49)."""
    M, K, N = 8192, 4096, 4096
    s49 = stl.strassen_rank49()
    g = torch.Generator(device=DEV).manual_seed(7)
    x = torch.randn((M, K), device=DEV, generator=g).to(torch.bfloat16)
    gy = torch.randn((M, N), device=DEV, generator=g).to(torch.bfloat16)
    w = (torch.randn((K, N), device=DEV, generator=g) / 64.0).to(torch.bfloat16)
    w_enc = stl.encode_tiles(w.float(), s49.on(x.device).e_w, 4).to(torch.bfloat16)
    layer = stl.StlLayer(s49, w_enc)
    _, cache = stl._layer_forward_cached(layer, x)
    g_x = stl._layer_backward(layer, cache, gy)[3]
    ref = gy.float() @ w.float().T
    assert rel(g_x.float(), ref) <= BF16_TOL


# ----------------------------------------------------------------- errors / edge cases
def test_errors_match_reference_classes():
    snf = stl.SnfTriple(4, 8, np.ones((8, 16)), np.ones((8, 16)), np.ones((8, 16)))
    with pytest.raises(stl.ShapeError):
        stl.stl_batched(torch.ones((6, 8), device=DEV), torch.zeros((2, 2, 8)), snf)
    with pytest.raises(stl.ShapeError):
        stl.stl_batched(torch.ones((8, 8), device=DEV), torch.zeros((2, 2, 7)), snf)
    with pytest.raises(ValueError):
        stl.encode_tiles(torch.tensor([[float("nan")] * 4] * 4, device=DEV), np.ones((8, 16)), 4)
    with pytest.raises(IndexError):
        stl.extract_slice(torch.zeros((2, 2, 3)), 3)
    layer = stl.StlLayer(snf, torch.zeros((2, 2, 8)))
    with pytest.raises(stl.ShapeError):
        stl.stl_layer_forward(layer, torch.ones((6, 8), device=DEV))
    with pytest.raises(stl.ShapeError):
        stl.SnfTriple(4, 8, np.ones((8, 16)), np.ones((8, 16)), np.ones((8, 15)))


def test_edge_cases():
    # scalar degeneration t = r = 1 equals matmul (test_snf_operator.py:75-79)
    one = np.ones((1, 1))
    unit = stl.SnfTriple(1, 1, one, one, one)
    rng = O.make_rng(4)
    x = rng.standard_normal((5, 7))
    w = rng.standard_normal((7, 3))
    got = stl.stl_reference(torch.tensor(x, dtype=torch.float32, device=DEV),
                            torch.tensor(w, dtype=torch.float32), unit)
    assert rel(got, x @ w) <= FP32_TOL
    # zero left factor gives exact zeros
    snf = stl.random_gaussian_init(4, 20, O.make_rng(6))
    out = stl.stl_reference(torch.zeros((8, 8), device=DEV), torch.randn((8, 8)), snf)
    assert bool((out == 0).all())
    # empty batch
    layer = stl.StlLayer(snf, torch.zeros((2, 3, 20)))
    y = stl.stl_layer_forward(layer, torch.zeros((0, 8), device=DEV))
    assert tuple(y.shape) == (0, 12)
    # identity encoder round trip (test_snf_operator.py:64-67)
    m = torch.randn((8, 8), device=DEV)
    enc = stl.encode_tiles(m, np.eye(16), 4)
    assert torch.equal(stl.decode_tiles(enc, np.eye(16), 4), m)


# ----------------------------------------------------------------- tensor-core transforms
@pytest.mark.parametrize("M,K,N,r", [(1024, 512, 768, 24), (512, 2048, 256, 32), (256, 64, 128, 7),
                                     (1040, 528, 1072, 16), (1024, 512, 1024, 24)])
def test_transform_paths_and_product_formats(M, K, N, r):
    """The t=4 transform paths (streaming kernels; the mma / register fallbacks where the tile
    columns are not multiples of 64) and every slice-product format the shape allows (fp32,
    F24, bf16) agree with each other and with the oracle, forward and backward."""
    t = 4
    rng = O.make_rng(3 * M + r)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    x_dev, x64 = bf16_round(rng.standard_normal((M, K)))
    w_dev, w64 = bf16_round(O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t))
    gy_dev, gy64 = bf16_round(rng.standard_normal((M, N)))
    layer = stl.StlLayer(stl.SnfTriple(t, r, e_x, e_w, d), w_dev)
    outs = {}
    for prod in (torch.float32, "f24", None):
        try:
            stl.cache_format(M, K, N, t, r, torch.bfloat16, prod)
        except ValueError:
            continue
        y, cache = stl._layer_forward_cached(layer, x_dev, products=prod)
        y_enc = stl.unpack_slice_products(cache.y_enc, r, M // t, N // t)
        outs[str(prod)] = (y, cache.u, y_enc) + tuple(stl._layer_backward(layer, cache, gy_dev))
    torch.cuda.synchronize()
    y_ref, cache_ref = O.layer_forward_cached(x64, w64, e_x, d, t)
    refs = (y_ref, cache_ref[1].transpose(2, 0, 1), cache_ref[2].transpose(2, 0, 1)) + \
        tuple(O.layer_backward(w64, e_x, d, cache_ref, gy64, t))
    names = ("y", "u", "y_enc", "g_ex", "g_d", "g_w", "g_x")
    base = outs[str(torch.float32)]
    for i, name in enumerate(names):
        for key, out in outs.items():
            # bf16 slice products round y_enc / g_u once more (2^-9) than fp32-class formats
            assert rel(out[i], base[i]) <= (5e-3 if key == "None" else 3e-3), (name, key)
            assert rel(out[i], refs[i]) <= BF16_TOL, (name, key, rel(out[i], refs[i]))


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [0, 32])
def test_inference_forward_product_formats(bits):
    """Cache-less bf16 forward with bf16 slice products (default) and with forced F24 ones,
    both against the float64 restatement on the same bf16 inputs (bar 1e-2)."""
    from paper_2503_12211_b200.snf_operator import _forward

    dev = torch.device("cuda")
    M, K, N, t, r = 1024, 768, 1536, 4, 24
    snf = stl.random_gaussian_init(t, r, stl.make_rng(3), scale=0.5).to(dev)
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
    w0 = torch.randn((K, N), device=dev, generator=g) / K ** 0.5
    w = stl.weights_to_planes(stl.encode_tiles(w0, snf.e_w, t).float(), dtype=torch.bfloat16)
    xt = x.double().reshape(M // t, t, K // t, t).permute(0, 2, 1, 3).reshape(M // t, K // t, t * t)
    prod = torch.einsum("ikp,pjk->ijp", xt @ snf.e_x.double().T, w.double())
    yref = (prod @ snf.d.double()).reshape(M // t, N // t, t, t).permute(0, 2, 1, 3).reshape(M, N)
    y = _forward(x, w, snf, products="f24" if bits else None)
    err = float((y.double() - yref).norm() / yref.norm())
    assert err < 1e-2 and err < (4e-3 if bits == 0 else 3.5e-3), err


# ----------------------------------------------------------------- fused chain (f1)
def test_three_layer_chain_strassen49_fp32():
    """Mirror of the reference's test_three_layer_chain_with_strassen
    (test_snf_operator.py:185-195): Strassen-49 is exact, so encode -> products -> 2 fused steps
    -> decode equals x W0 W1 W2 (fp32 path, generic remix since r > 32)."""
    e_x, e_w, d = O.strassen_rank49()
    s49 = stl.SnfTriple(4, 49, e_x, e_w, d)
    rng = O.make_rng(18)
    n = 256
    x = rng.standard_normal((n, n))
    ws = [rng.standard_normal((n, n)) / np.sqrt(n) for _ in range(3)]
    expected = x @ ws[0] @ ws[1] @ ws[2]
    encs = [torch.tensor(O.encode_tiles(w, e_w, 4), dtype=torch.float32) for w in ws]
    h = stl._slice_products(stl.encode_tiles(torch.tensor(x, dtype=torch.float32, device="cuda"),
                                             s49.e_x, 4), encs[0])
    for enc in encs[1:]:
        h = stl.stl_fused_step(h, enc, s49)
    got = stl.decode_tiles(h, s49.d, 4)
    assert rel(got, expected) <= FP32_TOL


@pytest.mark.parametrize("r,n", [(24, 512), (13, 256), (32, 768)])
def test_chain_bf16_streamed_remix(r, n):
    """A bf16 chain kept in 2-byte planes: bf16 products -> stl_fused_step (streaming remix,
    bf16 out) x 2 -> decode, against the oracle chain on the same bf16 weights (bar 1e-2)."""
    t = 4
    rng = O.make_rng(100 + r)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.5)
    snf = stl.SnfTriple(t, r, e_x, e_w, d)
    x_dev, x64 = bf16_round(rng.standard_normal((n, n)))
    w_dev, w64 = [], []
    for _ in range(3):
        a, b = bf16_round(O.encode_tiles(rng.standard_normal((n, n)) / np.sqrt(n), e_w, t))
        w_dev.append(a.cuda())
        w64.append(b)
    h = stl._slice_products(stl.encode_tiles(x_dev.cuda(), snf.e_x, t), w_dev[0]).to(torch.bfloat16)
    h64 = O.slice_products(O.encode_tiles(x64, e_x, t), w64[0])
    for wd, w6 in zip(w_dev[1:], w64[1:]):
        h = stl.stl_fused_step(h, wd, snf)
        assert h.dtype == torch.bfloat16
        h64 = O.stl_fused_step(h64, w6, e_x, d)
    got = stl.decode_tiles(h, snf.d, t)
    assert rel(got, O.decode_tiles(h64, d, t)) <= BF16_TOL
