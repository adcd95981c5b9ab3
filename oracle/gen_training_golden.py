"""Golden vectors for the Class-0 trainer and fake-encoding machinery,
computed by the REFERENCE (strassen_tile.training).

Run in the build container (where /root/reference is mounted):

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_training_golden.py

Writes tests/golden/training/training.json: training runs (configs, loss curves, best
factors, divergence outcomes), closed-form and Monte Carlo losses, per-pair gradients, and
a solution matrix with its per-W regression, each from the reference's own functions on
seeded inputs. The test re-draws the same inputs from the same seeds.
"""

from __future__ import annotations

import json
import sys
from dataclasses import asdict
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "training"

RUNS = [
    dict(r=24, seed=0, steps=300),
    dict(r=16, init="random_gaussian", seed=1, steps=200, init_scale=0.5, optimizer="plain_sgd",
         step_size=0.01),
    dict(r=24, seed=2, steps=300, fixed_w_population=True, n_train_pairs=512),
    dict(r=20, seed=3, steps=60, eval_every=7, plateau_patience=1, step_size=0.02, batch=64),
    dict(r=49, seed=0, steps=100),
    dict(r=8, init="random_gaussian", seed=4, steps=600, eval_every=10, plateau_patience=2,
         batch=64, step_size=0.05, init_scale=0.3),
    dict(r=16, init="random_gaussian", seed=0, steps=2000, step_size=75.0, init_scale=0.5,
         optimizer="plain_sgd"),
]


def main() -> None:
    sys.path.insert(0, str(REF))
    from strassen_tile import dense_core, strassen_basis, training

    out = {"runs": []}
    for kw in RUNS:
        cfg = training.Class0Config(**kw)
        rec = {"config": asdict(cfg)}
        try:
            res, tri = training.train_class0(cfg)
            rec["result"] = json.loads(res.to_json())
            rec["factors"] = [tri.e_x.tolist(), tri.e_w.tolist(), tri.d.tolist()]
        except training.DivergenceError as err:
            rec["divergence"] = {"message": str(err), "curve": err.curve}
        out["runs"].append(rec)

    # losses: population closed form and a Monte Carlo batch for a seeded Gaussian triple
    snf = strassen_basis.random_gaussian_init(4, 12, dense_core.make_rng(2), scale=0.5)
    rng = dense_core.make_rng(3)
    xs, ws = rng.standard_normal((2000, 4, 4)), rng.standard_normal((2000, 4, 4))
    out["losses"] = {"population": training.population_class0_loss(snf),
                     "monte_carlo": training.class0_loss(snf, list(zip(xs, ws)))}
    # per-pair gradients
    rng = dense_core.make_rng(5)
    snf = strassen_basis.random_gaussian_init(4, 14, rng, scale=0.5)
    pair = (rng.standard_normal((4, 4)), rng.standard_normal((4, 4)))
    out["gradients"] = [g.tolist() for g in training.class0_gradients(snf, pair)]
    # solution matrix, per-W regression and fake-encoding loss
    rng = dense_core.make_rng(10)
    snf = strassen_basis.random_gaussian_init(4, 20, rng, scale=0.6)
    xs = rng.standard_normal((100, 4, 4))
    w = rng.standard_normal((4, 4))
    f = training.solution_matrix(snf.e_x, snf.d, xs)
    fe = f @ w.reshape(-1)
    out["fake_encoding"] = {
        "solution": f.tolist(),
        "regression": training.per_w_fake_encoding_regression(snf.e_x, snf.d, w, xs).tolist(),
        "loss": training.fake_encoding_loss(snf.e_x, snf.d, fe, w, xs),
    }
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / "training.json").write_text(json.dumps(out, indent=None, sort_keys=True))


if __name__ == "__main__":
    main()
