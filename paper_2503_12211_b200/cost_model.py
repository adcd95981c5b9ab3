"""Algorithmic FLOP / byte accounting for the STL hot path (roofline denominators).

Restates the closed forms of ``strassen_tile.cost_model`` (cost_model.py:68-124) — one MAC is
2 FLOPs; square forms assume pre-encoded weights — and adds the byte counts of the B200
kernels actually launched, which is what bench.py divides by time.
"""

from __future__ import annotations

from dataclasses import dataclass

FLOPS_PER_MAC = 2


def flops_general(n: int, k: int, m: int, t: int, r: int) -> int:
    """Three transform passes + slice products (cost_model.py:68-78)."""
    per_tile = FLOPS_PER_MAC * t * t * r
    transforms = ((n * k) // (t * t) + (m * k) // (t * t) + (m * n) // (t * t)) * per_tile
    return transforms + FLOPS_PER_MAC * r * (n * k * m) // (t ** 3)


def flops_square(n: int, t: int, r: int) -> tuple[int, int]:
    """(STL, naive) FLOPs, pre-encoded weights (cost_model.py:81-91)."""
    return 2 * FLOPS_PER_MAC * n * n * r + FLOPS_PER_MAC * r * n ** 3 // t ** 3, FLOPS_PER_MAC * n ** 3


def io_square(n: int, t: int, r: int, bytes_per_scalar: int = 2):
    """(STL bytes, naive bytes, per-step breakdown) (cost_model.py:94-110)."""
    x = n * n * bytes_per_scalar
    sl = bytes_per_scalar * (n // t) ** 2 * r
    io1, io2, io3 = x + sl, 3 * sl, x + sl
    return io1 + io2 + io3, 3 * x, (io1, io2, io3)


def io_fused_chain(n: int, t: int, r: int, layers: int, bytes_per_scalar: int = 2) -> int:
    """Chain of layers with interior decode+encode fused (cost_model.py:113-124)."""
    if layers < 1:
        raise ValueError(f"need at least one layer, got {layers}")
    total, _, (io1, _, io3) = io_square(n, t, r, bytes_per_scalar)
    return layers * total - (layers - 1) * (io1 + io3)


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
