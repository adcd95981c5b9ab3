"""The Strassen-Tile (STL) operator on B200 — drop-in mirror of ``strassen_tile.snf_operator``.

Same names, argument order and error classes as the reference
(/root/reference/pkg/src/strassen_tile/snf_operator.py); the arithmetic runs in the sm_100a
kernels of ``libstl_b200.so`` through the C ABI (include/stl_b200.h):

==========================  =====================================  ==========================
reference (file:line)       this module                            C entry point
==========================  =====================================  ==========================
SnfTriple       :45-70      SnfTriple (fp32 factors on the GPU)    —
encode_tiles    :80-85      encode_tiles                           stl_encode
decode_tiles    :88-96      decode_tiles                           stl_decode
extract_slice   :99-104     extract_slice                          — (a view)
_slice_products :107-116    _slice_products                        stl_slice_gemm
stl_reference   :119-153    stl_reference (same map, GPU path)     stl_encode + stl_forward
stl_batched     :156-172    stl_batched                            stl_forward
stl_fused_step  :175-188    stl_fused_step                         stl_fused_step
==========================  =====================================  ==========================

Differences a caller can observe (documented in DESIGN.md §boundary):

* Encoded tensors are returned in the reference's (rows, cols, r) shape as zero-copy views of
  slice-major GPU planes (r, rows, cols); pass them back unchanged and no copy happens.
* Arithmetic is fp32 (fp32 in -> fp32 out, FFMA) or bf16 (bf16 in -> bf16 out, tcgen05 with
  fp32 accumulation and fp32 slice accumulators); f64 input is computed in fp32.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .dense_core import ShapeError, as_matrix, default_device, to_tensor


def _dt(dtype: torch.dtype) -> int:
    if dtype == torch.bfloat16:
        return _lib.STL_BF16
    if dtype == torch.float32:
        return _lib.STL_F32
    raise ValueError(f"unsupported compute dtype {dtype}")


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _coef(a, name: str, device: torch.device) -> torch.Tensor:
    """Encoder/decoder factor as a contiguous fp32 (r, t*t) device tensor."""
    m = to_tensor(a, device=device, dtype=torch.float32)
    if m.ndim != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={m.ndim}")
    return m.contiguous()


@dataclass
class SnfTriple:
    """Encoder/encoder/decoder triple with tile size t and rank r (snf_operator.py:45-70).

    All three factors are r x t^2 fp32 tensors (kept on the GPU once ``to()`` is called or the
    triple is first used); the decoder acts as d.T. r <= t^2 is legal.
    """

    t: int
    r: int
    e_x: torch.Tensor
    e_w: torch.Tensor
    d: torch.Tensor

    def __post_init__(self):
        if self.t < 1 or self.r < 1:
            raise ShapeError(f"need t >= 1 and r >= 1, got t={self.t}, r={self.r}")
        want = (self.r, self.t * self.t)
        for name in ("e_x", "e_w", "d"):
            v = getattr(self, name)
            m = v if isinstance(v, torch.Tensor) else torch.as_tensor(v, dtype=torch.float64)
            m = m.to(dtype=torch.float32)
            if m.ndim != 2 or tuple(m.shape) != want:
                raise ShapeError(f"{name} must be {want}, got {tuple(m.shape)}")
            if m.numel() and not bool(torch.isfinite(m).all()):
                raise ValueError(f"{name} contains non-finite entries")
            setattr(self, name, m.contiguous())

    def copy(self) -> "SnfTriple":
        return SnfTriple(self.t, self.r, self.e_x.clone(), self.e_w.clone(), self.d.clone())

    def to(self, device) -> "SnfTriple":
        """Move the factors to ``device`` in place; returns self."""
        for name in ("e_x", "e_w", "d"):
            setattr(self, name, getattr(self, name).to(device).contiguous())
        return self

    def on(self, device: torch.device) -> "SnfTriple":
        if self.e_x.device != device:
            self.to(device)
        return self

    @classmethod
    def from_reference(cls, snf) -> "SnfTriple":
        """Wrap any object with t, r, e_x, e_w, d (e.g. a numpy ``strassen_tile.SnfTriple``)."""
        return cls(int(snf.t), int(snf.r), snf.e_x, snf.e_w, snf.d)


def as_triple(snf) -> SnfTriple:
    return snf if isinstance(snf, SnfTriple) else SnfTriple.from_reference(snf)


def _check_encoded(enc, name: str = "encoded", device=None, dtype=None) -> torch.Tensor:
    e = to_tensor(enc, device=device, dtype=dtype)
    if e.ndim != 3:
        raise ShapeError(f"{name} must be a (block_rows, block_cols, r) tensor")
    return e


def _planes(enc: torch.Tensor) -> torch.Tensor:
    """(R, C, r) reference-shaped tensor -> contiguous slice-major planes (r, R, C)."""
    p = enc.permute(2, 0, 1)
    return p if p.is_contiguous() else p.contiguous()


def _weight_planes(w_enc: torch.Tensor) -> tuple[torch.Tensor, int]:
    """(bk, bj, r) encoded weights -> (planes, layout) without copying when possible.

    (r, bj, bk) storage (this package's native layout) is the K-major B operand; (r, bk, bj)
    storage (a permuted reference array) is used as the MN-major B operand.
    """
    kmaj = w_enc.permute(2, 1, 0)
    if kmaj.is_contiguous():
        return kmaj, _lib.STL_K_MAJOR
    mn = w_enc.permute(2, 0, 1)
    if mn.is_contiguous():
        return mn, _lib.STL_MN_MAJOR
    return kmaj.contiguous(), _lib.STL_K_MAJOR


def weights_to_planes(w_encoded, dtype: torch.dtype | None = None, device=None) -> torch.Tensor:
    """Reference-layout encoded weights (bk, bj, r) -> native K-major planes (r, bj, bk)."""
    w = _check_encoded(w_encoded, "w_encoded", device=device, dtype=dtype)
    return w.permute(2, 1, 0).contiguous()


def planes_to_weights(planes: torch.Tensor) -> torch.Tensor:
    """Native planes (r, bj, bk) -> reference-layout view (bk, bj, r)."""
    return planes.permute(2, 1, 0)


def encode_tiles(m, encoder, t: int) -> torch.Tensor:
    """Per-tile encoding: out[I, J, :] = encoder @ vec_tile(m, I, J, t) (snf_operator.py:80-85)."""
    m = as_matrix(m, "m")
    enc = _coef(encoder, "encoder", m.device)
    if enc.shape[1] != t * t:
        raise ShapeError(f"encoder needs {t * t} columns, got {enc.shape[1]}")
    if t < 1 or m.shape[0] % t or m.shape[1] % t:
        raise ShapeError(f"tile size {t} does not divide shape {tuple(m.shape)}")
    r = enc.shape[0]
    out = torch.empty((r, m.shape[0] // t, m.shape[1] // t), dtype=m.dtype, device=m.device)
    _lib.check(_lib.load().stl_encode(
        m.data_ptr(), _dt(m.dtype), m.shape[0], m.shape[1], m.stride(0), enc.data_ptr(), t, r,
        out.data_ptr(), _dt(out.dtype), _stream(m.device)))
    return out.permute(1, 2, 0)


def decode_tiles(enc, decoder, t: int) -> torch.Tensor:
    """Per-tile decoding with the transposed decoder (snf_operator.py:88-96)."""
    enc = _check_encoded(enc)
    dec = _coef(decoder, "decoder", enc.device)
    if tuple(dec.shape) != (enc.shape[2], t * t):
        raise ShapeError(f"decoder must be {(enc.shape[2], t * t)}, got {tuple(dec.shape)}")
    planes = _planes(enc)
    r, br, bc = planes.shape
    out = torch.empty((br * t, bc * t), dtype=enc.dtype, device=enc.device)
    _lib.check(_lib.load().stl_decode(
        planes.data_ptr(), _dt(planes.dtype), br, bc, r, dec.data_ptr(), t, out.data_ptr(),
        _dt(out.dtype), out.stride(0), _stream(enc.device)))
    return out


def extract_slice(enc, p: int) -> torch.Tensor:
    """The (block_rows x block_cols) matrix of p-th coordinates (snf_operator.py:99-104)."""
    enc = _check_encoded(enc)
    if not 0 <= p < enc.shape[2]:
        raise IndexError(f"slice index {p} out of range for rank {enc.shape[2]}")
    return enc[:, :, p].contiguous()


def _slice_products(x_enc, w_enc) -> torch.Tensor:
    """All r slice matmuls: out[:, :, p] = x_enc[:, :, p] @ w_enc[:, :, p] (:107-116).

    bf16 x bf16 runs the tcgen05 tensor-core kernel; anything else runs in fp32 (FFMA).
    The result is fp32 (the slice accumulators are never rounded to bf16).
    """
    x_enc = _check_encoded(x_enc, "x_enc")
    w_enc = _check_encoded(w_enc, "w_enc", device=x_enc.device)
    if x_enc.shape[2] != w_enc.shape[2]:
        raise ShapeError(f"rank mismatch: {x_enc.shape[2]} vs {w_enc.shape[2]}")
    if x_enc.shape[1] != w_enc.shape[0]:
        raise ShapeError(
            f"block grids incompatible: {tuple(x_enc.shape[:2])} x {tuple(w_enc.shape[:2])}")
    ab = torch.bfloat16 if (x_enc.dtype == torch.bfloat16 and w_enc.dtype == torch.bfloat16) \
        else torch.float32
    a = _planes(x_enc.to(ab))
    b, b_layout = _weight_planes(w_enc.to(ab))
    r, bi, bk = a.shape
    bj = w_enc.shape[1]
    out = torch.empty((r, bi, bj), dtype=torch.float32, device=x_enc.device)
    _lib.check(_lib.load().stl_slice_gemm(
        a.data_ptr(), _lib.STL_K_MAJOR, b.data_ptr(), b_layout, out.data_ptr(), _lib.STL_F32,
        _dt(ab), r, bi, bj, bk, _stream(x_enc.device)))
    return out.permute(1, 2, 0)


def forward_scratch(M: int, K: int, N: int, t: int, r: int, dtype: torch.dtype,
                    device: torch.device) -> torch.Tensor:
    """Device workspace for stl_forward (from the torch caching allocator, stream-safe)."""
    nbytes = int(_lib.load().stl_forward_scratch_bytes(M, K, N, t, r, _dt(dtype)))
    return torch.empty((max(nbytes, 1),), dtype=torch.uint8, device=device)


def _prod(products) -> int:
    """Slice-product format argument: None = per shape (STL_PROD_AUTO), or torch.bfloat16 /
    "f24" / torch.float32 to force one (include/stl_b200.h)."""
    if products is None:
        return _lib.STL_PROD_AUTO
    if products == "f24":
        return _lib.STL_F24
    return _dt(products)


def cache_format(M: int, K: int, N: int, t: int, r: int, dtype: torch.dtype, products=None) -> int:
    """Format of the y_enc cache a training forward writes (stl_cache_format): STL_F32,
    STL_BF16 or STL_F24; ValueError when the forced `products` format cannot be used."""
    f = int(_lib.load().stl_cache_format(M, K, N, t, r, _dt(dtype), _prod(products)))
    if f < 0:
        _lib.check(2)
    return f


def cache_bytes(M: int, K: int, N: int, t: int, r: int, dtype: torch.dtype, products=None) -> int:
    """Bytes of the forward cache y_enc (stl_cache_bytes_ex)."""
    return int(_lib.load().stl_cache_bytes_ex(M, K, N, t, r, _dt(dtype), _prod(products)))


def cache_dtype_format(y_enc: torch.Tensor) -> int:
    """The format a y_enc cache tensor holds — the cache carries it in its dtype: uint8 = F24
    bytes, bfloat16 = bf16 planes, float32 = fp32 planes."""
    if y_enc.dtype == torch.uint8:
        return _lib.STL_F24
    return _dt(y_enc.dtype)


def unpack_slice_products(y_enc: torch.Tensor, r: int, rows: int, cols: int) -> torch.Tensor:
    """fp32 planes (r, rows, cols) of a y_enc cache in any of its formats.

    uint8 caches are F24: the high 16 bits of every element, then the next 8 bits (bf16 path,
    see include/stl_b200.h stl_cache_bytes); plane caches are fp32 or bf16.
    """
    if y_enc.dtype != torch.uint8:
        return y_enc.float().reshape(r, rows, cols)
    n = r * rows * cols
    hi = y_enc[: 2 * n].view(torch.int16).to(torch.int32) & 0xFFFF
    lo = y_enc[2 * n: 3 * n].to(torch.int32)
    return ((hi << 16) | (lo << 8)).view(torch.float32).reshape(r, rows, cols)


def _forward(x: torch.Tensor, w_planes: torch.Tensor, snf: SnfTriple, keep_cache: bool = False,
             products=None):
    """Shared forward launch: returns y (and the (u, y_enc) cache when keep_cache).

    y_enc is fp32 planes (fp32 mode), or on the bf16 path bf16 planes or a uint8 F24 buffer
    (cache_format decides; the tensor's dtype records it for the backward);
    unpack_slice_products gives fp32 planes for any of them. `products`: see _prod."""
    t, r = snf.t, snf.r
    M, K = x.shape
    if w_planes.dtype != x.dtype:
        raise ValueError(f"weights dtype {w_planes.dtype} != input dtype {x.dtype}")
    if w_planes.ndim != 3 or w_planes.shape[0] != r:
        raise ShapeError(f"weight planes must be (r={r}, N/t, K/t), got {tuple(w_planes.shape)}")
    bk, bj = w_planes.shape[2], w_planes.shape[1]
    if bk * t != K:
        raise ShapeError(f"x tiling {(M // t, K // t)} incompatible with weights {(bk, bj)}")
    N = bj * t
    dev = x.device
    snf.on(dev)
    prod = _prod(products)
    u = torch.empty((r, M // t, bk), dtype=x.dtype, device=dev)
    y_enc = None
    if keep_cache:
        fmt = cache_format(M, K, N, t, r, x.dtype, products)
        if fmt == _lib.STL_F24:
            y_enc = torch.empty((3 * r * (M // t) * bj,), dtype=torch.uint8, device=dev)
        else:
            y_enc = torch.empty((r, M // t, bj),
                                dtype=torch.bfloat16 if fmt == _lib.STL_BF16 else torch.float32,
                                device=dev)
    y = torch.empty((M, N), dtype=x.dtype, device=dev)
    scratch = forward_scratch(M, K, N, t, r, x.dtype, dev)
    _lib.check(_lib.load().stl_forward_ex(
        x.data_ptr(), M, K, x.stride(0), w_planes.data_ptr(), N, snf.e_x.data_ptr(),
        snf.d.data_ptr(), t, r, _dt(x.dtype), y.data_ptr(), y.stride(0), u.data_ptr(),
        y_enc.data_ptr() if y_enc is not None else None, scratch.data_ptr(), scratch.numel(),
        prod, _stream(dev)))
    return (y, u, y_enc) if keep_cache else y


def stl_batched(x, w_encoded, snf) -> torch.Tensor:
    """Encode x, r slice-wise matmuls, decode (snf_operator.py:156-172)."""
    snf = as_triple(snf)
    x = as_matrix(x, "x")
    w = _check_encoded(w_encoded, "w_encoded", device=x.device, dtype=x.dtype)
    if w.shape[2] != snf.r:
        raise ShapeError(f"encoded rank {w.shape[2]} != triple rank {snf.r}")
    t = snf.t
    if x.shape[0] % t or x.shape[1] % t:
        raise ShapeError(f"tile size {t} does not divide shape {tuple(x.shape)}")
    if x.shape[1] // t != w.shape[0]:
        raise ShapeError(
            f"x tiling {(x.shape[0] // t, x.shape[1] // t)} incompatible with weights "
            f"{tuple(w.shape[:2])}")
    planes = w.permute(2, 1, 0)
    if not planes.is_contiguous():
        planes = planes.contiguous()
    return _forward(x, planes, snf)


def stl_reference(x, w, snf) -> torch.Tensor:
    """The reference's ground-truth map (snf_operator.py:119-153) evaluated on the GPU path.

    Encodes the raw weight matrix with e_w, then applies the batched operator. The loop-shaped
    CPU evaluation itself lives in oracle/ (test infrastructure), not in the product.
    """
    snf = as_triple(snf)
    x = as_matrix(x, "x")
    w = as_matrix(w, "w", dtype=x.dtype, device=x.device)
    t = snf.t
    if x.shape[1] != w.shape[0]:
        raise ShapeError(f"inner dims differ: {tuple(x.shape)} x {tuple(w.shape)}")
    for m, name in ((x, "x"), (w, "w")):
        if m.shape[0] % t or m.shape[1] % t:
            raise ShapeError(f"tile size {t} does not divide {name} shape {tuple(m.shape)}")
    return stl_batched(x, encode_tiles(w, snf.on(x.device).e_w, t), snf)


def stl_fused_step(x_encoded_prev, w_encoded, snf) -> torch.Tensor:
    """One fused layer step in encoded space (snf_operator.py:175-188, Algorithm 2).

    fp32 (or f64 / numpy) x_encoded_prev -> fp32 slice products (the reference contract). A
    bf16 x_encoded_prev with bf16 weights keeps a bf16 chain in 2-byte planes end to end: the
    remix is the streaming tensor-core kernel and the products come back bf16
    (stl_fused_step_ex)."""
    snf = as_triple(snf)
    bf16_chain = isinstance(x_encoded_prev, torch.Tensor) and x_encoded_prev.dtype == torch.bfloat16
    x_prev = _check_encoded(x_encoded_prev, "x_encoded_prev",
                            dtype=None if bf16_chain else torch.float32)
    dtype = torch.bfloat16 if (isinstance(w_encoded, torch.Tensor)
                               and w_encoded.dtype == torch.bfloat16) else torch.float32
    if bf16_chain and dtype != torch.bfloat16:
        raise ValueError("a bf16 encoded activation needs bf16 encoded weights")
    w = _check_encoded(w_encoded, "w_encoded", device=x_prev.device, dtype=dtype)
    if x_prev.shape[2] != snf.r or w.shape[2] != snf.r:
        raise ShapeError("encoded ranks must equal the triple rank")
    if x_prev.shape[1] != w.shape[0]:
        raise ShapeError(
            f"block grids incompatible: {tuple(x_prev.shape[:2])} x {tuple(w.shape[:2])}")
    dev = x_prev.device
    snf.on(dev)
    r = snf.r
    xp = _planes(x_prev)
    _, br, bk = xp.shape
    bj = w.shape[1]
    wp = w.permute(2, 1, 0)
    if not wp.is_contiguous():
        wp = wp.contiguous()
    out_dtype = torch.bfloat16 if bf16_chain else torch.float32
    out = torch.empty((r, br, bj), dtype=out_dtype, device=dev)
    mixed = torch.empty((r, br, bk), dtype=dtype, device=dev)
    comp = torch.empty((r, r), dtype=torch.float32, device=dev)
    _lib.check(_lib.load().stl_fused_step_ex(
        xp.data_ptr(), _dt(xp.dtype), br, bk, wp.data_ptr(), bj, snf.e_x.data_ptr(),
        snf.d.data_ptr(), snf.t, r, _dt(dtype), out.data_ptr(), _dt(out_dtype), mixed.data_ptr(),
        comp.data_ptr(), _stream(dev)))
    return out.permute(1, 2, 0)
