"""CPU oracle for the STL hot path — TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference's algorithm (arXiv 2503.12211 reference package,
/root/reference/pkg/src/strassen_tile). Each function cites the reference file:line it
restates. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this module — as the checker or the timed CPU baseline, never as the product
path (the product is paper_2503_12211_b200/, which has no CPU fallback).

Parity pinning: tests/test_oracle_golden.py checks every function below against golden
vectors produced by running the reference itself in the build container
(oracle/gen_golden.py -> tests/golden/*.npz), so this restatement is pinned to the
reference's own outputs, not only to self-consistency.
"""

from __future__ import annotations

import numpy as np


class ShapeError(ValueError):
    """dense_core.py:30-31."""


# ------------------------------------------------------------------ layout (dense_core.py)
def as_matrix(a, name="matrix"):
    """dense_core.py:42-49: finite, C-contiguous float64 2-D array."""
    m = np.ascontiguousarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={m.ndim}")
    if m.size and not np.isfinite(m).all():
        raise ValueError(f"{name} contains non-finite entries")
    return m


def tile_fibers(m, t):
    """dense_core.py:98-108: fiber[I, J, a*t + b] = m[I*t + a, J*t + b]."""
    m = as_matrix(m)
    R, C = m.shape
    if t < 1 or R % t or C % t:
        raise ShapeError(f"tile size {t} does not divide shape {m.shape}")
    return np.ascontiguousarray(np.transpose(m.reshape(R // t, t, C // t, t), (0, 2, 1, 3))
                                ).reshape(R // t, C // t, t * t)


def untile_fibers(f, t):
    """dense_core.py:111-119: inverse of tile_fibers."""
    f = np.asarray(f, dtype=np.float64)
    if f.ndim != 3 or f.shape[2] != t * t:
        raise ShapeError(f"expected (R, C, {t * t}) fibers, got {f.shape}")
    R, C, _ = f.shape
    return np.ascontiguousarray(np.transpose(f.reshape(R, C, t, t), (0, 2, 1, 3))
                                ).reshape(R * t, C * t)


# ------------------------------------------------------------------ operator (snf_operator.py)
def encode_tiles(m, encoder, t):
    """snf_operator.py:80-85: enc[I, J, p] = sum_c encoder[p, c] fiber[I, J, c]."""
    e = as_matrix(encoder, "encoder")
    if e.shape[1] != t * t:
        raise ShapeError(f"encoder needs {t * t} columns, got {e.shape[1]}")
    return np.einsum("ijc,pc->ijp", tile_fibers(m, t), e, optimize=True)


def decode_tiles(enc, decoder, t):
    """snf_operator.py:88-96: tile (I, J) = unvec(decoder^T enc[I, J, :])."""
    enc = np.asarray(enc, dtype=np.float64)
    d = as_matrix(decoder, "decoder")
    if enc.ndim != 3 or d.shape != (enc.shape[2], t * t):
        raise ShapeError("decoder/encoded shapes disagree")
    return untile_fibers(np.einsum("ijp,pc->ijc", enc, d, optimize=True), t)


def slice_products(x_enc, w_enc):
    """snf_operator.py:107-116: out[:, :, p] = x_enc[:, :, p] @ w_enc[:, :, p]."""
    x_enc = np.asarray(x_enc, dtype=np.float64)
    w_enc = np.asarray(w_enc, dtype=np.float64)
    if x_enc.shape[2] != w_enc.shape[2] or x_enc.shape[1] != w_enc.shape[0]:
        raise ShapeError("slice product shapes disagree")
    out = np.empty((x_enc.shape[0], w_enc.shape[1], x_enc.shape[2]))
    for p in range(x_enc.shape[2]):
        out[:, :, p] = x_enc[:, :, p] @ w_enc[:, :, p]
    return out


def stl_batched(x, w_encoded, e_x, d, t):
    """snf_operator.py:156-172: decode(slice_products(encode(x, e_x), w_enc), d)."""
    return decode_tiles(slice_products(encode_tiles(x, e_x, t), w_encoded), d, t)


def stl_reference_loop(x, w, e_x, e_w, d, t):
    """snf_operator.py:119-153: per-tile Hadamard accumulation over ascending L, decoded once.

    Pure-Python loops: use at small sizes only."""
    x = as_matrix(x, "x")
    w = as_matrix(w, "w")
    e_x, e_w, d = (as_matrix(a) for a in (e_x, e_w, d))
    r = e_x.shape[0]
    bi, bk, bj = x.shape[0] // t, x.shape[1] // t, w.shape[1] // t
    ux = np.array([[e_x @ x[i * t:(i + 1) * t, l * t:(l + 1) * t].reshape(-1)
                    for l in range(bk)] for i in range(bi)]).reshape(bi, bk, r)
    vw = np.array([[e_w @ w[l * t:(l + 1) * t, j * t:(j + 1) * t].reshape(-1)
                    for j in range(bj)] for l in range(bk)]).reshape(bk, bj, r)
    out = np.empty((x.shape[0], w.shape[1]))
    for i in range(bi):
        for j in range(bj):
            acc = np.zeros(r)
            for l in range(bk):
                acc += ux[i, l] * vw[l, j]
            out[i * t:(i + 1) * t, j * t:(j + 1) * t] = (d.T @ acc).reshape(t, t)
    return out


def stl_fused_step(x_encoded_prev, w_encoded, e_x, d):
    """snf_operator.py:175-188: slice_products(x_prev @ (e_x d^T)^T, w_enc)."""
    comp = as_matrix(e_x) @ as_matrix(d).T
    return slice_products(np.asarray(x_encoded_prev, dtype=np.float64) @ comp.T, w_encoded)


# ------------------------------------------------------------------ layer (toy_network.py)
def layer_forward_cached(x, weights, e_x, d, t):
    """toy_network.py:86-92: y and the cache (vx, u, y_enc)."""
    vx = tile_fibers(x, t)
    u = vx @ as_matrix(e_x).T
    y_enc = slice_products(u, weights)
    return untile_fibers(y_enc @ as_matrix(d), t), (vx, u, y_enc)


def layer_backward(weights, e_x, d, cache, gy, t):
    """toy_network.py:95-106: (g_ex, g_d, g_w, g_x), written with BLAS contractions."""
    vx, u, y_enc = cache
    weights = np.asarray(weights, dtype=np.float64)
    gvy = tile_fibers(gy, t)
    r = u.shape[2]
    g_d = np.einsum("ijp,ijc->pc", y_enc, gvy, optimize=True)
    g_enc = gvy @ as_matrix(d).T
    g_w = np.empty_like(weights)
    g_u = np.empty_like(u)
    for p in range(r):
        g_w[:, :, p] = u[:, :, p].T @ g_enc[:, :, p]
        g_u[:, :, p] = g_enc[:, :, p] @ weights[:, :, p].T
    g_ex = np.einsum("ikp,ikc->pc", g_u, vx, optimize=True)
    g_x = untile_fibers(g_u @ as_matrix(e_x), t)
    return g_ex, g_d, g_w, g_x


def layer_backward_einsum(weights, e_x, d, cache, gy, t):
    """toy_network.py:95-106 exactly as the reference evaluates it (np.einsum without
    `optimize`, which does not reach BLAS) — used only as the timed CPU baseline."""
    vx, u, y_enc = cache
    gvy = tile_fibers(gy, t)
    g_d = np.einsum("ijp,ijc->pc", y_enc, gvy)
    g_enc = gvy @ as_matrix(d).T
    g_w = np.einsum("ikp,ijp->kjp", u, g_enc)
    g_u = np.einsum("kjp,ijp->ikp", weights, g_enc)
    g_ex = np.einsum("ikp,ikc->pc", g_u, vx)
    g_x = untile_fibers(g_u @ as_matrix(e_x), t)
    return g_ex, g_d, g_w, g_x


def stl_batched_reference_numpy(x, w_encoded, e_x, d, t):
    """snf_operator.py:156-172 with the reference's own numpy call pattern (tile_fibers @ E.T,
    transposed batched np.matmul, enc @ d) — the timed CPU baseline of bench.py."""
    x_enc = tile_fibers(x, t) @ as_matrix(e_x).T
    w_enc = np.asarray(w_encoded, dtype=np.float64)
    prod = np.matmul(x_enc.transpose(2, 0, 1), w_enc.transpose(2, 0, 1)).transpose(1, 2, 0)
    return untile_fibers(np.ascontiguousarray(prod) @ as_matrix(d), t)


# ------------------------------------------------------------------ fixtures (strassen_basis.py)
_S7_A = np.array([[1, 0, 0, 1], [0, 0, 1, 1], [1, 0, 0, 0], [0, 0, 0, 1], [1, 1, 0, 0],
                  [-1, 0, 1, 0], [0, 1, 0, -1]], dtype=np.float64)   # strassen_basis.py:34-45
_S7_B = np.array([[1, 0, 0, 1], [1, 0, 0, 0], [0, 1, 0, -1], [-1, 0, 1, 0], [0, 0, 0, 1],
                  [1, 1, 0, 0], [0, 0, 1, 1]], dtype=np.float64)   # strassen_basis.py:46-57
_S7_D = np.array([[1, 0, 0, 1], [0, 0, 1, -1], [0, 1, 0, 1], [1, 0, 1, 0], [-1, 1, 0, 0],
                  [0, 0, 0, 1], [1, 0, 0, 0]], dtype=np.float64)   # strassen_basis.py:58-69


def strassen_rank49():
    """strassen_basis.py:77-129: kron(F, F) @ P_blockmajor for each factor."""
    perm = np.zeros((16, 16))
    for i in range(4):
        for j in range(4):
            perm[4 * (2 * (i // 2) + j // 2) + 2 * (i % 2) + (j % 2), 4 * i + j] = 1.0
    return tuple(np.kron(f, f) @ perm for f in (_S7_A, _S7_B, _S7_D))


def random_gaussian_init(t, r, rng, scale=1.0):
    """strassen_basis.py:155-168: (e_x, e_w, d) drawn in that order."""
    shape = (r, t * t)
    return tuple(scale * rng.standard_normal(shape) for _ in range(3))


def make_rng(seed):
    """dense_core.py:152-154."""
    return np.random.Generator(np.random.PCG64(seed))


def rel_frobenius(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / (den if den > 0 else 1.0))
