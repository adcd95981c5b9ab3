"""FLOP / IO accounting for the STL hot path: the reference's cost model + B200 kernel bytes.

Mirrors ``strassen_tile.cost_model`` (cost_model.py:1-195) name for name — ``ProblemShape``,
``CostReport``, ``flops_general``, ``flops_square``, ``io_square``, ``io_fused_chain``,
``cost_report``, ``count_reference_flops``, ``speedup_table`` — with the same conventions (one
MAC = 2 FLOPs; square forms assume pre-encoded weights; exact integer arithmetic) and the same
``ShapeError`` on invalid shapes. ``count_reference_flops`` runs this package's GPU pipeline
(encode -> slice GEMMs -> decode through the C ABI) and tallies the MACs of every executed
launch from the shapes it actually processed.

``LayerCost`` adds the byte counts of the B200 kernels actually launched, which
is what bench.py divides by time for the roofline fractions.
"""

from __future__ import annotations

from dataclasses import dataclass

from .dense_core import ShapeError

FLOPS_PER_MAC = 2


@dataclass(frozen=True)
class ProblemShape:
    """An n x k by k x m STL problem with tile size t and rank r (cost_model.py:27-41)."""

    n: int
    k: int
    m: int
    t: int
    r: int
    bytes_per_scalar: int = 2

    def __post_init__(self):
        dims = (self.n, self.k, self.m, self.t, self.r, self.bytes_per_scalar)
        if any(int(v) != v or v < 1 for v in dims):
            raise ShapeError(f"all shape fields must be positive integers: {self}")
        if self.n % self.t or self.k % self.t or self.m % self.t:
            raise ShapeError(f"tile size {self.t} must divide n, k, m in {self}")


@dataclass(frozen=True)
class CostReport:
    """Square-shape cost summary; steps 1/2/3 = encode / slice products / decode
    (cost_model.py:44-65). Totals equal the sums of their breakdowns."""

    n: int
    t: int
    r: int
    bytes_per_scalar: int
    flops_stl: int
    flops_naive: int
    io_stl_bytes: int
    io_naive_bytes: int
    flop_steps: tuple[int, int, int]
    io_steps: tuple[int, int, int]

    @property
    def speedup_flops(self) -> float:
        return self.flops_naive / self.flops_stl


def flops_general(shape: ProblemShape) -> int:
    """Three transform passes at 2 t^2 r FLOPs per tile + the slice products
    2 r n k m / t^3 (cost_model.py:68-78)."""
    n, k, m, t, r = shape.n, shape.k, shape.m, shape.t, shape.r
    per_tile = FLOPS_PER_MAC * t * t * r
    transforms = ((n * k) // (t * t) + (m * k) // (t * t) + (m * n) // (t * t)) * per_tile
    return transforms + FLOPS_PER_MAC * r * (n * k * m) // (t * t * t)


def flops_square(n: int, t: int, r: int) -> tuple[int, int]:
    """(STL, naive) FLOPs for n x n operands with pre-encoded weights (cost_model.py:81-91):
    4 n^2 r transform FLOPs + 2 n^3 r / t^3, against 2 n^3."""
    ProblemShape(n, n, n, t, r)  # validation, as the reference
    return (2 * FLOPS_PER_MAC * n * n * r + FLOPS_PER_MAC * r * n ** 3 // t ** 3,
            FLOPS_PER_MAC * n ** 3)


def io_square(n: int, t: int, r: int, bytes_per_scalar: int = 2):
    """(STL bytes, naive bytes, per-step STL breakdown) for square shapes (cost_model.py:94-110):
    step 1 reads X and writes r slices, step 2 reads both slice stacks and writes the products,
    step 3 mirrors step 1; naive matmul moves 3 |X|."""
    ProblemShape(n, n, n, t, r, bytes_per_scalar)
    x = n * n * bytes_per_scalar
    sl = bytes_per_scalar * (n // t) ** 2 * r
    io1, io2, io3 = x + sl, 3 * sl, x + sl
    return io1 + io2 + io3, 3 * x, (io1, io2, io3)


def io_fused_chain(n: int, t: int, r: int, layers: int, bytes_per_scalar: int = 2) -> int:
    """Chain of layers with interior decode+encode fused: each interior boundary saves an
    io3 + io1 pair (cost_model.py:113-124)."""
    if layers < 1:
        raise ShapeError(f"need at least one layer, got {layers}")
    total, _, (io1, _, io3) = io_square(n, t, r, bytes_per_scalar)
    return layers * total - (layers - 1) * (io1 + io3)


def cost_report(n: int, t: int, r: int, bytes_per_scalar: int = 2) -> CostReport:
    """The square-shape FLOP and IO closed forms in one report (cost_model.py:127-147)."""
    flops_stl, flops_naive = flops_square(n, t, r)
    each = FLOPS_PER_MAC * n * n * r
    io_stl, io_naive, io_steps = io_square(n, t, r, bytes_per_scalar)
    return CostReport(n=n, t=t, r=r, bytes_per_scalar=bytes_per_scalar, flops_stl=flops_stl,
                      flops_naive=flops_naive, io_stl_bytes=io_stl, io_naive_bytes=io_naive,
                      flop_steps=(each, flops_stl - 2 * each, each), io_steps=io_steps)


def count_reference_flops(shape: ProblemShape, seed: int = 0) -> int:
    """Run the batched pipeline on random data and tally executed MACs (cost_model.py:150-187).

    The reference counts inside its numpy loops; here the pipeline is this package's GPU path —
    encode X and W (stl_encode), the r slice GEMMs (stl_slice_gemm), decode (stl_decode) — and
    each launch adds the MACs of the tiles / slice products it returned, so the count is taken
    from what ran. It must equal ``flops_general(shape)``. Needs a GPU (no CPU fallback).
    """
    import torch

    from .dense_core import make_rng, to_tensor
    from .snf_operator import _slice_products, decode_tiles, encode_tiles
    from .strassen_basis import random_gaussian_init

    n, k, m, t, r = shape.n, shape.k, shape.m, shape.t, shape.r
    rng = make_rng(seed)
    x = to_tensor(rng.standard_normal((n, k)))
    w = to_tensor(rng.standard_normal((k, m)))
    snf = random_gaussian_init(t, r, rng, scale=0.5)
    flops = 0
    x_enc = encode_tiles(x, snf.e_x, t)
    flops += FLOPS_PER_MAC * r * t * t * x_enc.shape[0] * x_enc.shape[1]
    w_enc = encode_tiles(w, snf.e_w, t)
    flops += FLOPS_PER_MAC * r * t * t * w_enc.shape[0] * w_enc.shape[1]
    out_enc = _slice_products(x_enc, w_enc)
    flops += FLOPS_PER_MAC * out_enc.shape[2] * out_enc.shape[0] * out_enc.shape[1] * x_enc.shape[1]
    y = decode_tiles(out_enc, snf.d, t)
    flops += FLOPS_PER_MAC * r * t * t * (y.shape[0] // t) * (y.shape[1] // t)
    torch.cuda.synchronize()
    return flops


def speedup_table(n_list, r_list, t: int, bytes_per_scalar: int = 2) -> list[CostReport]:
    """Cost reports over the (n, r) grid, n-major then r (cost_model.py:190-195)."""
    return [cost_report(n, t, r, bytes_per_scalar) for n in n_list for r in r_list]


@dataclass(frozen=True)
class LayerCost:
    """Per-launch algorithmic work of one STL layer step, rectangular M x K x N."""

    M: int
    K: int
    N: int
    t: int
    r: int
    s: int = 2  # bytes per scalar of the compute dtype
    p: int = 4  # bytes per stored slice product (4 = fp32, 3 = F24 on the bf16 path)

    @property
    def bi(self):
        return self.M // self.t

    @property
    def bk(self):
        return self.K // self.t

    @property
    def bj(self):
        return self.N // self.t

    # --- FLOPs
    def gemm_flops(self) -> int:
        """One batch of r slice GEMMs (bi x bk) . (bk x bj)."""
        return FLOPS_PER_MAC * self.r * self.bi * self.bk * self.bj

    def dense_equiv_flops(self) -> int:
        """The dense GEMM the layer replaces: 2 M K N."""
        return FLOPS_PER_MAC * self.M * self.K * self.N

    def forward_flops(self) -> int:
        """encode + slice products + decode (flops_square generalised)."""
        return (FLOPS_PER_MAC * self.M * self.K * self.r + self.gemm_flops()
                + FLOPS_PER_MAC * self.M * self.N * self.r)

    def backward_flops(self) -> int:
        """encode(gY) + g_d + two slice GEMMs + decode(g_u) + g_ex."""
        return 2 * self.gemm_flops() + 2 * FLOPS_PER_MAC * self.r * (self.M * self.N + self.M * self.K)

    # --- bytes actually moved by the unfused kernels (each tensor read/written once)
    def encode_bytes(self) -> int:
        return self.M * self.K * self.s + self.r * self.bi * self.bk * self.s

    def gemm_fwd_bytes(self) -> int:
        return (self.r * self.bi * self.bk * self.s + self.r * self.bj * self.bk * self.s
                + self.r * self.bi * self.bj * self.p)

    def decode_bytes(self) -> int:
        return self.r * self.bi * self.bj * self.p + self.M * self.N * self.s

    def encode_gy_gd_bytes(self) -> int:
        """gY in, y_enc cache in, g_enc planes out (the g_d reduction rides along)."""
        return self.M * self.N * self.s + self.r * self.bi * self.bj * (self.p + self.s)

    def decode_gu_gex_bytes(self) -> int:
        """g_u products in, X in (for g_ex), g_x out."""
        return self.r * self.bi * self.bk * self.p + 2 * self.M * self.K * self.s

    def forward_min_bytes(self) -> int:
        """|X| + |W_enc| + |Y|: the fused lower bound."""
        return self.M * self.K * self.s + self.r * self.bj * self.bk * self.s + self.M * self.N * self.s
