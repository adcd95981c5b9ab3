"""Loaders for the committed golden fixtures (tests/golden/*.npz) — test infrastructure."""

from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent.parent / "tests" / "golden"


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def golden_cases(name: str) -> dict:
    """Group 'case/key' arrays of a golden file into {case: {key: array}}."""
    out: dict = {}
    for k, v in load_golden(name).items():
        case, key = k.split("/", 1)
        out.setdefault(case, {})[key] = v
    return out
