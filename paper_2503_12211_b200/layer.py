"""The STL layer (forward, cached forward, analytic backward) on B200.

Mirror of the hot-path part of ``strassen_tile.toy_network`` (toy_network.py:45-106):
``StlLayer``, ``stl_layer_forward``, ``_layer_forward_cached`` and ``_layer_backward`` keep the
reference's names, argument order, ShapeError checks and return conventions; the arithmetic is
``stl_forward_ex`` / ``stl_backward_ex`` of the C ABI (the cache's slice-product format is
recorded by its dtype and passed to the backward explicitly). On top of that, ``StlLinear`` packages the same
kernels as a ``torch.autograd.Function`` / ``nn.Module`` for training (the DP path of bench.py).

Weights are held in the native slice-major layout ``w_planes`` (r, out_tiles, in_tiles); the
``weights`` attribute is the reference-layout (in_tiles, out_tiles, r) zero-copy view.
"""

from __future__ import annotations

from typing import NamedTuple

import torch

from . import _lib
from .dense_core import ShapeError, as_matrix, to_tensor
from .snf_operator import SnfTriple, _dt, _forward, _stream, as_triple, cache_dtype_format


class StlLayer:
    """One tile-operator layer: trainable (e_x, d) plus fake-encoded weights (:45-71)."""

    def __init__(self, snf, weights, dtype: torch.dtype | None = None):
        self.snf = as_triple(snf)
        w = to_tensor(weights, dtype=dtype)
        if w.ndim != 3 or w.shape[2] != self.snf.r:
            raise ShapeError(
                f"weights must be (in_tiles, out_tiles, {self.snf.r}), got {tuple(w.shape)}")
        self.w_planes = w.permute(2, 1, 0).contiguous()
        self.snf.on(self.w_planes.device)

    @property
    def weights(self) -> torch.Tensor:
        return self.w_planes.permute(2, 1, 0)

    @weights.setter
    def weights(self, w) -> None:
        w = to_tensor(w, device=self.w_planes.device, dtype=self.w_planes.dtype)
        self.w_planes = w.permute(2, 1, 0).contiguous()

    @property
    def dtype(self) -> torch.dtype:
        return self.w_planes.dtype

    @property
    def in_dim(self) -> int:
        return self.w_planes.shape[2] * self.snf.t

    @property
    def out_dim(self) -> int:
        return self.w_planes.shape[1] * self.snf.t


class LayerCache(NamedTuple):
    """Forward state needed by the backward (toy_network.py:86-92).

    vx: the layer input itself (the reference keeps tile_fibers(x), the same numbers);
    u: encoded input planes (r, M/t, K/t) in the compute dtype;
    y_enc: slice products (r, M/t, N/t): fp32 planes in fp32 mode; on the bf16 path a uint8
    F24 buffer (24-bit slice products, see stl_cache_bytes) or bf16 planes.
    ``unpack_slice_products`` returns fp32 planes for any of them.
    """

    vx: torch.Tensor
    u: torch.Tensor
    y_enc: torch.Tensor


def _check_input(layer: StlLayer, x) -> torch.Tensor:
    x = as_matrix(x, "x", dtype=layer.dtype, device=layer.w_planes.device)
    t = layer.snf.t
    if x.shape[0] % t:
        raise ShapeError(f"batch {x.shape[0]} not divisible by tile size {t}")
    if x.shape[1] != layer.in_dim:
        raise ShapeError(f"input width {x.shape[1]} != layer in_dim {layer.in_dim}")
    return x


def stl_layer_forward(layer: StlLayer, x) -> torch.Tensor:
    """Batched layer application; rows of x are samples (toy_network.py:74-83)."""
    x = _check_input(layer, x)
    return _forward(x, layer.w_planes, layer.snf)


def _layer_forward_cached(layer: StlLayer, x, *, products=None):
    """Forward plus the (vx, u, y_enc) cache (toy_network.py:86-92).

    `products` (keyword, not in the reference): force the slice-product format of the cache
    (torch.bfloat16, "f24", torch.float32; default per shape, include/stl_b200.h)."""
    x = _check_input(layer, x)
    y, u, y_enc = _forward(x, layer.w_planes, layer.snf, keep_cache=True, products=products)
    return y, LayerCache(x, u, y_enc)


def backward_raw(snf: SnfTriple, w_planes: torch.Tensor, cache: LayerCache, gy: torch.Tensor,
                 need_gx: bool = True, need_gw: bool = True, need_enc: bool = True,
                 gw_ready: torch.cuda.Event | None = None):
    """Launch stl_backward_ex; returns (g_ex, g_d, g_w planes (r, bj, bk) fp32, g_x).
    gw_ready: an event recorded once g_w is final (before the g_x / g_ex decode)."""
    x, u, y_enc = cache
    t, r = snf.t, snf.r
    M, K = x.shape
    N = gy.shape[1]
    dev = x.device
    bi, bk, bj = M // t, K // t, N // t
    g_enc = torch.empty((r, bi, bj), dtype=x.dtype, device=dev)
    g_w = torch.empty((r, bj, bk), dtype=torch.float32, device=dev) if need_gw else None
    g_ex = torch.empty((r, t * t), dtype=torch.float32, device=dev) if need_enc else None
    g_d = torch.empty((r, t * t), dtype=torch.float32, device=dev) if need_enc else None
    g_x = torch.empty((M, K), dtype=x.dtype, device=dev) if (need_gx or need_enc) else None
    g_u = torch.empty((r, bi, bk), dtype=torch.float32, device=dev) if g_x is not None else None
    lib = _lib.load()
    red = torch.empty((int(lib.stl_reduce_workspace_floats(r, t)),), dtype=torch.float32,
                      device=dev) if need_enc else None

    def ptr(tns):
        return tns.data_ptr() if tns is not None else None

    if gw_ready is not None and not gw_ready.cuda_event:
        gw_ready.record()  # torch creates events lazily: materialise the handle
    # the cache carries its format (its dtype); the backward is told, never guesses
    _lib.check(lib.stl_backward_ex(
        gy.data_ptr(), gy.stride(0), x.data_ptr(), x.stride(0), w_planes.data_ptr(),
        snf.e_x.data_ptr(), snf.d.data_ptr(), u.data_ptr(), y_enc.data_ptr(),
        cache_dtype_format(y_enc), M, K, N, t, r, _dt(x.dtype), ptr(g_ex), ptr(g_d), ptr(g_w),
        ptr(g_x), K, g_enc.data_ptr(), ptr(g_u), ptr(red), _lib.STL_PROD_AUTO,
        gw_ready.cuda_event if gw_ready is not None else None, _stream(dev)))
    return g_ex, g_d, g_w, g_x


def _layer_backward(layer: StlLayer, cache, gy):
    """Gradients (g_ex, g_d, g_weights, g_x) for one layer (toy_network.py:95-106).

    g_weights is returned in the reference layout (in_tiles, out_tiles, r) as an fp32 view.
    """
    x = cache[0]
    gy = as_matrix(gy, "gy", dtype=x.dtype, device=x.device)
    if gy.shape != (x.shape[0], layer.out_dim):
        raise ShapeError(f"gy must be {(x.shape[0], layer.out_dim)}, got {tuple(gy.shape)}")
    g_ex, g_d, g_w, g_x = backward_raw(layer.snf, layer.w_planes, LayerCache(*cache), gy)
    return g_ex, g_d, g_w.permute(2, 1, 0), g_x


class StlLinearFunction(torch.autograd.Function):
    """y = STL(x; e_x, d, W_enc) with the fused-kernel backward. e_w gets no gradient."""

    @staticmethod
    def forward(ctx, x, w_planes, e_x, d, t: int, r: int):
        snf = _TripleView(t, r, e_x, d)
        y, u, y_enc = _forward(x, w_planes, snf, keep_cache=True)
        ctx.save_for_backward(x, u, y_enc, w_planes, e_x, d)
        ctx.tr = (t, r)
        return y

    @staticmethod
    def backward(ctx, gy):
        x, u, y_enc, w_planes, e_x, d = ctx.saved_tensors
        t, r = ctx.tr
        gy = gy.contiguous()
        need_gx, need_gw = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        need_enc = ctx.needs_input_grad[2] or ctx.needs_input_grad[3]
        g_ex, g_d, g_w, g_x = backward_raw(_TripleView(t, r, e_x, d), w_planes,
                                           LayerCache(x, u, y_enc), gy, need_gx, need_gw,
                                           need_enc)
        if g_w is not None and g_w.dtype != w_planes.dtype:
            g_w = g_w.to(w_planes.dtype)
        return (g_x if need_gx else None, g_w, g_ex if ctx.needs_input_grad[2] else None,
                g_d if ctx.needs_input_grad[3] else None, None, None)


class _TripleView:
    """Minimal triple (t, r, e_x, d) for the autograd path; factors already on the device."""

    def __init__(self, t, r, e_x, d):
        self.t, self.r, self.e_x, self.d = t, r, e_x.contiguous(), d.contiguous()

    def on(self, device):
        return self


class StlLinear(torch.nn.Module):
    """nn.Module form of an STL layer: parameters e_x, d (fp32) and w_planes (compute dtype).

    ``y = layer(x)`` for x of shape (M, in_dim) with M divisible by t; e_w is a buffer used only
    to build initial fake encodings (toy_network.py:241-252).
    """

    def __init__(self, snf, weights_planes: torch.Tensor):
        super().__init__()
        snf = as_triple(snf)
        self.t, self.r = snf.t, snf.r
        dev = weights_planes.device
        self.e_x = torch.nn.Parameter(snf.e_x.to(dev).clone())
        self.d = torch.nn.Parameter(snf.d.to(dev).clone())
        self.register_buffer("e_w", snf.e_w.to(dev).clone())
        self.w_planes = torch.nn.Parameter(weights_planes.contiguous())

    @classmethod
    def from_layer(cls, layer: StlLayer) -> "StlLinear":
        return cls(layer.snf, layer.w_planes)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if x.ndim != 2 or x.shape[0] % self.t or x.shape[1] != self.w_planes.shape[2] * self.t:
            raise ShapeError(f"input {tuple(x.shape)} incompatible with STL layer "
                             f"(t={self.t}, in_dim={self.w_planes.shape[2] * self.t})")
        if self.w_planes.ndim != 3 or self.w_planes.shape[0] != self.r:
            raise ShapeError(f"w_planes must be (r={self.r}, N/t, K/t), "
                             f"got {tuple(self.w_planes.shape)}")
        # the kernels compute in the weights' dtype (e.g. fp32 activations under a bf16 layer,
        # or autocast output): cast the input, never reinterpret its bytes
        if x.dtype != self.w_planes.dtype:
            x = x.to(self.w_planes.dtype)
        return StlLinearFunction.apply(x.contiguous(), self.w_planes, self.e_x, self.d, self.t,
                                       self.r)
