"""Trained-encoder source: the Class-0 trainer and the fake-encoding machinery.

Mirrors ``strassen_tile.training`` (reference training.py) with the same names, config fields,
RNG streams and error classes, so a triple trained here is the one the reference would train
(to f64 rounding) and drops straight into ``StlLayer`` / ``StlLinear``:

=========================================  =====================================================
reference (training.py)                    here
=========================================  =====================================================
Class0Config / Class0Result  :49-92        same dataclasses, same validation and JSON
_batch_loss / class0_loss    :103-118      one batched residual on the device
population_class0_loss       :121-139      closed form, batched over the rank
class0_gradients             :142-168      per-pair analytic gradients
_batch_gradients             :171-187      batched analytic gradients
train_class0                 :199-273      same loop; steps run in chunks of ``eval_every``
build_zw_vectors             :279-301      same
_zw_moments / solution_matrix :304-345     moments in closed form (Hadamard of two Grams)
fake_encoding_loss           :348-368      same
per_w_fake_encoding_regression :371-388    stacked regression, normal equations
init_toy_network (toy_network.py:239-250)  init_stl_layers: fake encodings of Gaussian weights
class0_base_triple (toy_network.py:253-258) same
=========================================  =====================================================

This math is tiny (r x t^2 factors, batches of t x t tiles) and is not the STL hot path: it
runs as float64 torch ops on the operator's device (the GPU by default; ``device=`` accepts any
torch device). Batches are drawn from the reference's numpy PCG64 streams (``spawn_rngs``) in
the reference's order and copied over once per chunk of ``eval_every`` steps. Per-step batch
losses stay on the device and are checked for divergence once per chunk — the divergence
checks only read losses, and the step size only changes at evaluations (chunk ends), so the
chunked loop takes exactly the reference's decisions: a divergence at step s inside a chunk
raises with the curve as it stood at step s.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from .dense_core import SINGULAR_COND_LIMIT, ShapeError, SingularSystemError, default_device
from .dense_core import spawn_rngs  # noqa: F401  (re-exported; dense_core.py:157-160)
from .snf_operator import SnfTriple, encode_tiles
from .strassen_basis import strassen_rank49

INIT_STRASSEN = "strassen_subset"
INIT_RANDOM = "random_gaussian"

DIVERGENCE_FACTOR = 10.0
DIVERGENCE_PATIENCE = 100
DIVERGENCE_FLOOR = 1e-9


class DivergenceError(RuntimeError):
    """Training loss blew past the divergence threshold; carries the curve (training.py:40-46)."""

    def __init__(self, message: str, curve: list[tuple[int, float]]):
        super().__init__(message)
        self.curve = curve


@dataclass
class Class0Config:
    """training.py:49-79 (same fields, defaults and validation)."""

    r: int
    t: int = 4
    init: str = INIT_STRASSEN
    seed: int = 0
    steps: int = 12000
    batch: int = 512
    step_size: float = 0.05
    optimizer: str = "momentum"  # or "plain_sgd"
    momentum: float = 0.9
    init_scale: float = 0.1
    n_train_pairs: int = 8192  # population size when fixed_w_population is set
    n_eval_pairs: int = 4096
    fixed_w_population: bool = False
    eval_every: int = 50
    plateau_patience: int = 8  # evals without improvement before halving the step
    min_step_size: float = 1e-4

    def validate(self) -> "Class0Config":
        if self.r < 1 or self.t < 1:
            raise ValueError(f"need r >= 1 and t >= 1, got r={self.r}, t={self.t}")
        if self.init not in (INIT_STRASSEN, INIT_RANDOM):
            raise ValueError(f"unknown init kind {self.init!r}")
        if self.optimizer not in ("plain_sgd", "momentum"):
            raise ValueError(f"unknown optimizer {self.optimizer!r}")
        counts = (self.steps, self.batch, self.n_train_pairs, self.n_eval_pairs, self.eval_every)
        if any(c < 1 for c in counts):
            raise ValueError(f"all counts must be positive: {self}")
        if self.step_size <= 0:
            raise ValueError(f"step_size must be > 0, got {self.step_size}")
        return self


@dataclass
class Class0Result:
    """training.py:82-92."""

    r: int
    init: str
    seed: int
    loss_init: float
    loss_final: float
    loss_curve: list[tuple[int, float]] = field(repr=False)

    def to_json(self) -> str:
        return json.dumps(asdict(self), sort_keys=True)


# ------------------------------------------------------------------ helpers
def _device(device) -> torch.device:
    return torch.device(device) if device is not None else default_device()


def _f64(a, dev: torch.device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.detach().to(device=dev, dtype=torch.float64)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(dev)


def _factors(snf, dev: torch.device):
    """(t, e_x, e_w, d) of any triple-like object, float64 on `dev`."""
    return int(snf.t), _f64(snf.e_x, dev), _f64(snf.e_w, dev), _f64(snf.d, dev)


def _matrix64(a, name: str, dev: torch.device) -> torch.Tensor:
    m = _f64(a, dev)
    if m.ndim != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={m.ndim}")
    if m.numel() and not bool(torch.isfinite(m).all()):
        raise ValueError(f"{name} contains non-finite entries")
    return m


def _stack_pairs(pairs, t: int, dev: torch.device):
    """training.py:95-100: a sequence of (X, W) t x t pairs -> (xs, ws) stacks."""
    pairs = list(pairs)
    if not pairs:
        raise ShapeError("need at least one (X, W) pair")
    if all(not isinstance(x, torch.Tensor) and not isinstance(w, torch.Tensor) for x, w in pairs):
        xs = _f64(np.stack([np.asarray(x, dtype=np.float64) for x, _ in pairs]), dev)
        ws = _f64(np.stack([np.asarray(w, dtype=np.float64) for _, w in pairs]), dev)
    else:
        xs = torch.stack([_f64(x, dev) for x, _ in pairs])
        ws = torch.stack([_f64(w, dev) for _, w in pairs])
    if tuple(xs.shape[1:]) != (t, t) or tuple(ws.shape[1:]) != (t, t):
        raise ShapeError(f"pairs must be {t}x{t} tiles, got {tuple(xs.shape[1:])} / "
                         f"{tuple(ws.shape[1:])}")
    if not (bool(torch.isfinite(xs).all()) and bool(torch.isfinite(ws).all())):
        raise ValueError("pairs contain non-finite entries")
    return xs, ws


def _residual(ex, ew, d, xs, ws):
    """(u, v, e) of a batch: u = vec(X) e_x^T, v = vec(W) e_w^T, e = vec(XW) - (u*v) d."""
    b, t2 = xs.shape[0], ex.shape[1]
    vx, vw = xs.reshape(b, t2), ws.reshape(b, t2)
    y = torch.bmm(xs, ws).reshape(b, t2)
    u = vx @ ex.T
    v = vw @ ew.T
    return vx, vw, u, v, y - (u * v) @ d


def _loss_dev(ex, ew, d, xs, ws) -> torch.Tensor:
    """training.py:103-111, as a 0-d device tensor."""
    e = _residual(ex, ew, d, xs, ws)[4]
    return (e * e).sum(dim=1).mean() / ex.shape[1]


def _grads_dev(ex, ew, d, xs, ws):
    """training.py:171-187."""
    vx, vw, u, v, e = _residual(ex, ew, d, xs, ws)
    scale = -2.0 / (ex.shape[1] * xs.shape[0])
    g_d = scale * ((u * v).T @ e)
    de = e @ d.T
    g_ex = scale * ((de * v).T @ vx)
    g_ew = scale * ((de * u).T @ vw)
    return g_ex, g_ew, g_d


# ------------------------------------------------------------------ losses and gradients
def class0_loss(snf, pairs, device=None) -> float:
    """Mean over (X, W) pairs of the per-entry squared matmul residual (training.py:114-118)."""
    dev = _device(device)
    t, ex, ew, d = _factors(snf, dev)
    xs, ws = _stack_pairs(pairs, t, dev)
    return float(_loss_dev(ex, ew, d, xs, ws))


def population_class0_loss(snf, device=None) -> float:
    """Exact expected loss over i.i.d. N(0,1) tile pairs, in closed form (training.py:121-139):
    (t^3 - 2 * sum_p <d_p, e_x,p e_w,p> + sum(G)) / t^2 with G the Hadamard product of the three
    factor Grams."""
    dev = _device(device)
    t, ex, ew, d = _factors(snf, dev)
    r = ex.shape[0]
    gram = (d @ d.T) * (ex @ ex.T) * (ew @ ew.T)
    cross = (d.reshape(r, t, t) * torch.bmm(ex.reshape(r, t, t), ew.reshape(r, t, t))).sum()
    return float((t ** 3 - 2.0 * cross + gram.sum()) / (t * t))


def class0_gradients(snf, pair, device=None):
    """Analytic per-pair gradients (g_ex, g_ew, g_d) of the residual (training.py:142-168)."""
    dev = _device(device)
    t, ex, ew, d = _factors(snf, dev)
    x, w = pair
    x, w = _matrix64(x, "x", dev), _matrix64(w, "w", dev)
    if tuple(x.shape) != (t, t) or tuple(w.shape) != (t, t):
        raise ShapeError(f"pair must be {t}x{t} tiles")
    g_ex, g_ew, g_d = _grads_dev(ex, ew, d, x[None], w[None])
    return g_ex, g_ew, g_d


# ------------------------------------------------------------------ trainer
def _initial_factors(cfg: Class0Config, rng: np.random.Generator, dev: torch.device):
    """training.py:190-196 in float64, drawing from `rng` exactly as the reference does
    (strassen_basis.py:132-137 row subset / :155-168 Gaussian factors)."""
    if cfg.init == INIT_STRASSEN:
        if cfg.t != 4:
            raise ValueError("strassen_subset initialization requires t=4")
        full = strassen_rank49()
        if not 1 <= cfg.r <= full.r:
            raise ValueError(f"subset rank must be in [1, {full.r}], got {cfg.r}")
        rows = torch.from_numpy(np.sort(rng.choice(full.r, size=cfg.r, replace=False)))
        return [_f64(f, dev)[rows.to(dev)].contiguous() for f in (full.e_x, full.e_w, full.d)]
    shape = (cfg.r, cfg.t * cfg.t)
    return [_f64(cfg.init_scale * rng.standard_normal(shape), dev) for _ in range(3)]


def _draw_chunk(cfg: Class0Config, rng: np.random.Generator, n: int, dev: torch.device,
                pool=None):
    """The next n steps' batches, drawn in the reference's order (training.py:222-228)."""
    t = cfg.t
    if pool is not None:
        idx = np.stack([rng.integers(0, cfg.n_train_pairs, size=cfg.batch) for _ in range(n)])
        idx = torch.from_numpy(idx).to(dev)
        return pool[0][idx], pool[1][idx]
    xs = np.empty((n, cfg.batch, t, t))
    ws = np.empty((n, cfg.batch, t, t))
    for i in range(n):
        xs[i] = rng.standard_normal((cfg.batch, t, t))
        ws[i] = rng.standard_normal((cfg.batch, t, t))
    return _f64(xs, dev), _f64(ws, dev)


def train_class0(cfg: Class0Config, device=None) -> tuple[Class0Result, SnfTriple]:
    """Minibatch gradient descent on the tile-matmul residual (training.py:199-273).

    Fresh Gaussian pairs per batch by default (``fixed_w_population`` resamples one fixed
    draw). The reported final loss is the held-out loss of the best checkpoint seen; that
    checkpoint is returned as an ``SnfTriple`` (fp32 factors, ready for the GPU operator; the
    float64 factors are attached as ``triple.factors64``). Deterministic given the config.
    """
    cfg.validate()
    dev = _device(device)
    init_rng, data_rng, eval_rng = spawn_rngs(cfg.seed, 3)
    t = cfg.t
    params = _initial_factors(cfg, init_rng, dev)

    eval_x = _f64(eval_rng.standard_normal((cfg.n_eval_pairs, t, t)), dev)
    eval_w = _f64(eval_rng.standard_normal((cfg.n_eval_pairs, t, t)), dev)
    pool = None
    if cfg.fixed_w_population:
        pool = (_f64(data_rng.standard_normal((cfg.n_train_pairs, t, t)), dev),
                _f64(data_rng.standard_normal((cfg.n_train_pairs, t, t)), dev))

    loss_init = float(_loss_dev(*params, eval_x, eval_w))
    curve: list[tuple[int, float]] = [(0, loss_init)]
    best_loss, best = loss_init, [p.clone() for p in params]
    diverge_threshold = DIVERGENCE_FACTOR * loss_init + DIVERGENCE_FLOOR
    diverged_streak = 0
    step_size = cfg.step_size
    since_improved = 0
    vel = [torch.zeros_like(p) for p in params]
    momentum = cfg.optimizer == "momentum"

    step = 0
    while step < cfg.steps:
        n = min(cfg.eval_every - step % cfg.eval_every, cfg.steps - step)
        bxs, bws = _draw_chunk(cfg, data_rng, n, dev, pool)
        losses = torch.empty(n, dtype=torch.float64, device=dev)
        for i in range(n):
            grads = _grads_dev(*params, bxs[i], bws[i])
            for k in range(3):
                if momentum:
                    vel[k].mul_(cfg.momentum).add_(grads[k])
                    params[k].sub_(step_size * vel[k])
                else:
                    params[k].sub_(step_size * grads[k])
            losses[i] = _loss_dev(*params, bxs[i], bws[i])
        for i, batch_loss in enumerate(losses.tolist()):
            s = step + i + 1
            if not np.isfinite(batch_loss):
                raise DivergenceError(f"non-finite loss at step {s}", curve)
            diverged_streak = diverged_streak + 1 if batch_loss > diverge_threshold else 0
            if diverged_streak >= DIVERGENCE_PATIENCE:
                raise DivergenceError(
                    f"loss above {DIVERGENCE_FACTOR}x the initial level for "
                    f"{DIVERGENCE_PATIENCE} consecutive steps at step {s}",
                    curve,
                )
        step += n
        # chunks end exactly at the reference's evaluation steps
        eval_loss = float(_loss_dev(*params, eval_x, eval_w))
        curve.append((step, eval_loss))
        if eval_loss < best_loss:
            best_loss, best = eval_loss, [p.clone() for p in params]
            since_improved = 0
        else:
            since_improved += 1
            if since_improved >= cfg.plateau_patience and step_size > cfg.min_step_size:
                step_size = max(step_size * 0.5, cfg.min_step_size)
                since_improved = 0

    result = Class0Result(r=cfg.r, init=cfg.init, seed=cfg.seed, loss_init=loss_init,
                          loss_final=best_loss, loss_curve=curve)
    triple = SnfTriple(t, cfg.r, *best)
    triple.factors64 = tuple(best)
    return result, triple


# ------------------------------------------------------------------ fake encodings
def build_zw_vectors(x, i: int, e_x, d, device=None):
    """Coefficient vectors of output coordinate i as linear functionals (training.py:279-301):
    z . vec(W) = vec(XW)_i and z' . f = (d^T (e_x vec(X) * f))_i."""
    dev = _device(device)
    x, e_x, d = _matrix64(x, "x", dev), _matrix64(e_x, "e_x", dev), _matrix64(d, "d", dev)
    t = x.shape[0]
    if tuple(x.shape) != (t, t) or e_x.shape[1] != t * t or d.shape != e_x.shape:
        raise ShapeError("x must be t x t and e_x, d must be r x t^2")
    if not 0 <= i < t * t:
        raise IndexError(f"coordinate {i} out of range for t^2 = {t * t}")
    a, b = divmod(i, t)
    z = torch.zeros(t * t, dtype=torch.float64, device=dev)
    z[b::t] = x[a, :]
    z_prime = d[:, i] * (e_x @ x.reshape(-1))
    return z, z_prime


def _samples(x_samples, t: int, dev: torch.device) -> torch.Tensor:
    xs = _f64(x_samples, dev)
    if xs.ndim != 3 or tuple(xs.shape[1:]) != (t, t) or xs.shape[0] < 1:
        raise ShapeError(f"x_samples must be a nonempty stack of {t}x{t} tiles")
    return xs


def _zw_moments(e_x, d, x_samples, dev: torch.device):
    """Empirical (E[z'z'^T], E[z'z^T]) over samples and uniform output coordinates
    (training.py:304-327), in closed form: with U = X_vec e_x^T,
      E[z'z'^T] = (U^T U) o (d d^T) / (S t^2)
      E[z'z^T][p, l t + b] = sum_a d[p, a t + b] * (sum_s U[s, p] X_s[a, l]) / (S t^2)."""
    e_x, d = _matrix64(e_x, "e_x", dev), _matrix64(d, "d", dev)
    r, t2 = e_x.shape
    t = int(round(t2 ** 0.5))
    xs = _samples(x_samples, t, dev)
    if t * t != t2 or d.shape != e_x.shape:
        raise ShapeError("e_x and d must be r x t^2")
    count = xs.shape[0] * t2
    u = xs.reshape(-1, t2) @ e_x.T  # (S, r)
    a = (u.T @ u) * (d @ d.T) / count
    q = torch.einsum("sp,sal->pal", u, xs)  # (r, t, t)
    bmat = torch.einsum("pab,pal->plb", d.reshape(r, t, t), q).reshape(r, t2) / count
    return a, bmat


def _check_cond(gram: torch.Tensor, what: str) -> None:
    cond = float(torch.linalg.cond(gram))
    if not np.isfinite(cond) or cond > SINGULAR_COND_LIMIT:
        raise SingularSystemError(f"{what} (cond ~ {cond:.3e})", cond=cond)


def solution_matrix(e_x, d, x_samples, device=None) -> torch.Tensor:
    """The r x t^2 map F sending vec(W) to its optimal fake encoding (training.py:330-345):
    F = E[z'z'^T]^{-1} E[z'z^T]."""
    dev = _device(device)
    a, bmat = _zw_moments(e_x, d, x_samples, dev)
    _check_cond(a, "fake-encoding Gram is numerically singular; more input samples or a "
                   "better-conditioned (e_x, d) needed")
    return torch.linalg.solve(a, bmat)


def fake_encoding_loss(e_x, d, fe, w, x_samples, device=None) -> float:
    """Empirical mean residual using a fixed fake encoding for W (training.py:348-368)."""
    dev = _device(device)
    e_x, d, w = _matrix64(e_x, "e_x", dev), _matrix64(d, "d", dev), _matrix64(w, "w", dev)
    fe = _f64(fe, dev).reshape(-1)
    t = w.shape[0]
    t2 = t * t
    if fe.shape[0] != e_x.shape[0]:
        raise ShapeError(f"fake encoding length {fe.shape[0]} != rank {e_x.shape[0]}")
    xs = _f64(x_samples, dev)
    if xs.ndim != 3 or tuple(xs.shape[1:]) != (t, t):
        raise ShapeError(f"x_samples must be a stack of {t}x{t} tiles")
    vx = xs.reshape(-1, t2)
    y = (xs @ w).reshape(-1, t2)
    resid = y - ((vx @ e_x.T) * fe) @ d
    return float((resid * resid).sum(dim=1).mean() / t2)


def per_w_fake_encoding_regression(e_x, d, w, x_samples, device=None) -> torch.Tensor:
    """Direct least-squares fake encoding for one W (training.py:371-388): one equation per
    sample and output coordinate, rows d[:, i] * (e_x vec(X)), solved by normal equations with
    the reference's singularity check (dense_core.py:122-141)."""
    dev = _device(device)
    e_x, d, w = _matrix64(e_x, "e_x", dev), _matrix64(d, "d", dev), _matrix64(w, "w", dev)
    t = w.shape[0]
    t2 = t * t
    xs = _samples(x_samples, t, dev)
    u = xs.reshape(-1, t2) @ e_x.T  # (S, r)
    rows = (u[:, None, :] * d.T[None, :, :]).reshape(-1, e_x.shape[0])  # (S t^2, r)
    targets = (xs @ w).reshape(-1)
    if rows.shape[0] < rows.shape[1]:
        raise ShapeError(f"underdetermined system: {rows.shape[0]} rows < {rows.shape[1]} cols")
    gram = rows.T @ rows
    _check_cond(gram, "rank-deficient Gram matrix")
    return torch.linalg.solve(gram, rows.T @ targets)


# ------------------------------------------------------------------ layer initialisation
def init_stl_layers(dims, base: SnfTriple, rng: np.random.Generator, dtype=None, device=None):
    """Fresh layers from a base triple (toy_network.py:239-250): each layer's weights are the
    fake encoding e_w . vec(W0) of a Gaussian W0 / sqrt(fan_in), encoded on the GPU."""
    from .layer import StlLayer

    dims = tuple(int(x) for x in dims)
    t = base.t
    if len(dims) < 2:
        raise ValueError("dims needs at least input and output widths")
    if any(x % t for x in dims):
        raise ValueError(f"layer widths {dims} must be divisible by t={t}")
    dev = _device(device)
    layers = []
    for i in range(len(dims) - 1):
        w0 = rng.standard_normal((dims[i], dims[i + 1])) / np.sqrt(dims[i])
        w0 = torch.from_numpy(w0).to(device=dev, dtype=dtype or torch.float32)
        snf = base.copy().to(dev)
        layers.append(StlLayer(snf, encode_tiles(w0, snf.e_w, t)))
    return layers


def class0_base_triple(r: int, t: int = 4, seed: int = 0, encoder_steps: int = 2000,
                       device=None) -> SnfTriple:
    """Weight-space triple from a quick synthetic-tile training run (toy_network.py:253-258)."""
    return train_class0(Class0Config(r=r, t=t, seed=seed, steps=encoder_steps, batch=256),
                        device=device)[1]
