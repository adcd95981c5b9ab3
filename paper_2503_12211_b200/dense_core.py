"""Host-side tensor conventions of the STL operator (torch mirror of the reference L1).

Mirrors the parts of ``strassen_tile.dense_core`` the hot path depends on:

* ``ShapeError`` — same class name and ``ValueError`` base (dense_core.py:30-31);
* ``as_matrix``  — coercion + non-finite rejection (dense_core.py:42-49), except that the GPU
  path computes in fp32 or bf16 instead of f64 (f64 input is cast to fp32);
* ``tile_fibers`` / ``untile_fibers`` / ``vec_tile`` / ``unvec_tile`` — the row-major t x t tile
  layout contract (dense_core.py:77-119). These are pure index permutations (torch views/copies);
  the kernels never materialise fibers, they read tiles straight from the row-major matrix;
* ``make_rng`` / ``spawn_rngs`` / ``gaussian_matrix`` — the seeded PCG64 streams the fixtures and
  benchmarks draw from (dense_core.py:152-166), bit-identical to the reference's.
"""

from __future__ import annotations

import numpy as np
import torch


class ShapeError(ValueError):
    """Operand shapes are incompatible or a matrix is not tileable."""


# Condition-number ceiling above which a normal-equation system counts as singular
# (dense_core.py:27).
SINGULAR_COND_LIMIT = 1e12


class SingularSystemError(ValueError):
    """A linear system is numerically singular; carries a condition estimate (dense_core.py:34-40)."""

    def __init__(self, message: str, cond: float | None = None):
        super().__init__(message)
        self.cond = cond


COMPUTE_DTYPES = (torch.float32, torch.bfloat16)

# The reference rejects non-finite inputs on every API call (dense_core.py:47-48). The check
# costs a device->host sync, so the training path (StlLinear) skips it; the flat function API
# keeps it on by default for drop-in behaviour. Toggle with set_check_finite().
_CHECK_FINITE = True


def set_check_finite(flag: bool) -> None:
    global _CHECK_FINITE
    _CHECK_FINITE = bool(flag)


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the STL operator runs on CUDA only (no CPU fallback); no GPU visible")
    return torch.device("cuda", torch.cuda.current_device())


def to_tensor(a, device: torch.device | None = None, dtype: torch.dtype | None = None) -> torch.Tensor:
    """numpy / torch / nested lists -> torch tensor on the CUDA device, compute dtype."""
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
    if dtype is None:
        dtype = t.dtype if t.dtype in COMPUTE_DTYPES else torch.float32
    dev = device if device is not None else (t.device if t.is_cuda else default_device())
    return t.to(device=dev, dtype=dtype)


def as_matrix(a, name: str = "matrix", dtype: torch.dtype | None = None,
              device: torch.device | None = None) -> torch.Tensor:
    """Coerce to a 2-D CUDA tensor with unit column stride (dense_core.py:42-49)."""
    m = to_tensor(a, device=device, dtype=dtype)
    if m.ndim != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={m.ndim}")
    if m.stride(1) != 1 or (m.shape[0] > 1 and m.stride(0) < m.shape[1]):
        m = m.contiguous()
    if _CHECK_FINITE and m.numel() and not bool(torch.isfinite(m).all()):
        raise ValueError(f"{name} contains non-finite entries")
    return m


def _check_tileable(shape, t: int) -> None:
    if t < 1:
        raise ShapeError(f"tile size must be >= 1, got {t}")
    if shape[0] % t or shape[1] % t:
        raise ShapeError(f"tile size {t} does not divide shape {tuple(shape)}")


def tile_fibers(m, t: int) -> torch.Tensor:
    """(rows/t, cols/t, t*t) fibers, fibers[I, J, :] = row-major vec of tile (I, J)."""
    m = to_tensor(m) if not isinstance(m, torch.Tensor) else m
    _check_tileable(m.shape, t)
    rows, cols = m.shape[0] // t, m.shape[1] // t
    return m.reshape(rows, t, cols, t).transpose(1, 2).reshape(rows, cols, t * t)


def untile_fibers(fibers, t: int) -> torch.Tensor:
    """Inverse of tile_fibers: (R, C, t*t) -> (R*t, C*t)."""
    f = fibers if isinstance(fibers, torch.Tensor) else to_tensor(fibers)
    if f.ndim != 3 or f.shape[2] != t * t:
        raise ShapeError(f"expected (R, C, {t * t}) fibers, got {tuple(f.shape)}")
    rows, cols = f.shape[0], f.shape[1]
    return f.reshape(rows, cols, t, t).transpose(1, 2).reshape(rows * t, cols * t)


def vec_tile(m, block_row: int, block_col: int, t: int) -> torch.Tensor:
    """Row-major flattening of one tile (dense_core.py:77-88)."""
    m = m if isinstance(m, torch.Tensor) else to_tensor(m)
    _check_tileable(m.shape, t)
    rows, cols = m.shape[0] // t, m.shape[1] // t
    if not (0 <= block_row < rows and 0 <= block_col < cols):
        raise ShapeError(f"tile index ({block_row},{block_col}) out of range for {rows}x{cols} grid")
    i, j = block_row * t, block_col * t
    return m[i : i + t, j : j + t].reshape(t * t).clone()


def unvec_tile(v, t: int) -> torch.Tensor:
    """Inverse of vec_tile: a length t*t vector back to a t x t tile (dense_core.py:90-95)."""
    v = (v if isinstance(v, torch.Tensor) else to_tensor(v)).reshape(-1)
    if v.shape[0] != t * t:
        raise ShapeError(f"expected length {t * t}, got {v.shape[0]}")
    return v.reshape(t, t).clone()


def make_rng(seed: int) -> np.random.Generator:
    """Seeded PCG64 generator; identical seeds give identical streams (dense_core.py:152-154)."""
    return np.random.Generator(np.random.PCG64(seed))


def spawn_rngs(seed: int, n: int) -> list[np.random.Generator]:
    """n independent child generators split deterministically from one seed
    (dense_core.py:157-160)."""
    seq = np.random.SeedSequence(seed)
    return [np.random.Generator(np.random.PCG64(child)) for child in seq.spawn(n)]


def gaussian_matrix(rng: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    """rows x cols matrix of i.i.d. standard normal entries (dense_core.py:163-167); host numpy,
    the same stream as the reference (move it to the GPU with ``to_tensor``)."""
    if rows < 1 or cols < 1:
        raise ShapeError(f"matrix dims must be >= 1, got {rows}x{cols}")
    return rng.standard_normal((rows, cols))
