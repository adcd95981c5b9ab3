"""Encoder fixtures for the STL operator (host side, numpy).

Same names, factor values and random streams as ``strassen_tile.strassen_basis``
(strassen_basis.py:21-168) so that a seeded run builds bit-identical triples:

* ``strassen_rank7``  — Strassen's 7-product 2x2 algorithm as an (e_x, e_w, d) triple (t=2);
* ``strassen_rank49`` — Strassen (x) Strassen for 4x4 tiles, conjugated from block-major to
  row-major vectorisation, with the exactness self-check over all 256 elementary pairs;
* ``pruned_subset_init`` / ``subset_triple`` — row subsets of a triple;
* ``random_gaussian_init`` — three i.i.d. N(0, scale^2) factors drawn in the order e_x, e_w, d.

These are CPU fixture providers ("stays on CPU"); the triples they return are
converted to GPU fp32 factors by :class:`~paper_2503_12211_b200.snf_operator.SnfTriple`.
"""

from __future__ import annotations

import numpy as np

from .dense_core import ShapeError, make_rng  # noqa: F401  (make_rng re-exported)
from .snf_operator import SnfTriple


class ConstructionError(RuntimeError):
    """The construction-time exactness self-check failed."""


# Strassen's products over row-major [m11, m12, m21, m22] coordinates:
#   M1 = (A11 + A22)(B11 + B22)   M2 = (A21 + A22) B11   M3 = A11 (B12 - B22)
#   M4 = A22 (B21 - B11)          M5 = (A11 + A12) B22   M6 = (A21 - A11)(B11 + B12)
#   M7 = (A12 - A22)(B21 + B22)
#   C11 = M1 + M4 - M5 + M7, C12 = M3 + M5, C21 = M2 + M4, C22 = M1 - M2 + M3 + M6
# e_x[p] holds the A coefficients of product p, e_w[p] the B coefficients, and d[p, c] the
# coefficient of product p in output entry c.
def _strassen_factors():
    a = np.zeros((7, 4))
    b = np.zeros((7, 4))
    c = np.zeros((7, 4))
    A11, A12, A21, A22 = range(4)
    prods = [
        ({A11: 1, A22: 1}, {A11: 1, A22: 1}),
        ({A21: 1, A22: 1}, {A11: 1}),
        ({A11: 1}, {A12: 1, A22: -1}),
        ({A22: 1}, {A21: 1, A11: -1}),
        ({A11: 1, A12: 1}, {A22: 1}),
        ({A21: 1, A11: -1}, {A11: 1, A12: 1}),
        ({A12: 1, A22: -1}, {A21: 1, A22: 1}),
    ]
    for p, (ca, cb) in enumerate(prods):
        for k, v in ca.items():
            a[p, k] = v
        for k, v in cb.items():
            b[p, k] = v
    outputs = {
        0: {0: 1, 3: 1, 4: -1, 6: 1},
        1: {2: 1, 4: 1},
        2: {1: 1, 3: 1},
        3: {0: 1, 1: -1, 2: 1, 5: 1},
    }
    for entry, terms in outputs.items():
        for p, v in terms.items():
            c[p, entry] = v
    return a, b, c


def strassen_rank7() -> SnfTriple:
    """Exact rank-7 triple for 2x2 tiles (t=2)."""
    a, b, c = _strassen_factors()
    return SnfTriple(2, 7, a, b, c)


def _rowmajor_to_blockmajor() -> np.ndarray:
    """P with P @ vec_rowmajor(4x4) = vec_blockmajor(4x4) (outer 2x2 block, then inner)."""
    p = np.zeros((16, 16))
    for i in range(4):
        for j in range(4):
            blk = 2 * (i // 2) + (j // 2)
            inner = 2 * (i % 2) + (j % 2)
            p[4 * blk + inner, 4 * i + j] = 1.0
    return p


def _bilinear_tensor(e_x, e_w, d) -> np.ndarray:
    return np.einsum("pa,pb,pc->abc", e_x, e_w, d)


def _matmul_tensor(t: int) -> np.ndarray:
    n = t * t
    out = np.zeros((n, n, n))
    for i in range(t):
        for k in range(t):
            for j in range(t):
                out[i * t + k, k * t + j, i * t + j] = 1.0
    return out


def strassen_rank49() -> SnfTriple:
    """Exact rank-49 triple for 4x4 tiles: kron(F, F) @ P for each factor, self-checked."""
    a, b, c = _strassen_factors()
    p = _rowmajor_to_blockmajor()
    e_x, e_w, d = (np.kron(f, f) @ p for f in (a, b, c))
    if not np.array_equal(_bilinear_tensor(e_x, e_w, d), _matmul_tensor(4)):
        raise ConstructionError("composed rank-49 triple failed the exactness check")
    return SnfTriple(4, 49, e_x, e_w, d)


def _np(snf: SnfTriple):
    return (snf.e_x.detach().cpu().double().numpy(), snf.e_w.detach().cpu().double().numpy(),
            snf.d.detach().cpu().double().numpy())


def pruned_subset_init(full: SnfTriple, r: int, rng: np.random.Generator) -> SnfTriple:
    """The same r rows (uniform, without replacement, sorted) of all three factors."""
    if not 1 <= r <= full.r:
        raise ValueError(f"subset rank must be in [1, {full.r}], got {r}")
    rows = np.sort(rng.choice(full.r, size=r, replace=False))
    ex, ew, d = _np(full)
    return SnfTriple(full.t, r, ex[rows], ew[rows], d[rows])


def subset_triple(full: SnfTriple, rows) -> SnfTriple:
    """Triple built from an explicit row subset (kept in the given order)."""
    rows = np.asarray(rows, dtype=int)
    if rows.ndim != 1 or rows.size < 1 or np.unique(rows).size != rows.size:
        raise ValueError("row subset must be a nonempty list of distinct indices")
    if rows.min() < 0 or rows.max() >= full.r:
        raise ValueError(f"row indices must lie in [0, {full.r})")
    ex, ew, d = _np(full)
    return SnfTriple(full.t, rows.size, ex[rows], ew[rows], d[rows])


def random_gaussian_init(t: int, r: int, rng: np.random.Generator, scale: float = 1.0) -> SnfTriple:
    """Three independent r x t^2 factors with i.i.d. N(0, scale^2) entries (e_x, e_w, d order)."""
    if t < 1 or r < 1:
        raise ShapeError(f"need t >= 1 and r >= 1, got t={t}, r={r}")
    shape = (r, t * t)
    e_x = scale * rng.standard_normal(shape)
    e_w = scale * rng.standard_normal(shape)
    d = scale * rng.standard_normal(shape)
    return SnfTriple(t, r, e_x, e_w, d)


def nested_subset_chain(rng: np.random.Generator, size: int = 49) -> np.ndarray:
    """A seeded permutation whose first-r prefixes form nested row subsets
    (strassen_basis.py:140-142)."""
    return rng.permutation(size)
