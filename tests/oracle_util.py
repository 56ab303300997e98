"""Shared helpers: build a golden case, replay its inputs, normwise error."""
from __future__ import annotations

import os

import numpy as np

from golden_cases import CASES
from paper_1503_02852_b200 import builders as B

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def case_net(name: str):
    spec = CASES[name]
    return getattr(B, spec["builder"])(*spec["args"], **spec.get("kwargs", {}))


def case_inputs(name: str, net):
    """Regenerate the per-iteration (x, target) pairs exactly as make_golden.py drew them."""
    spec = CASES[name]
    rng = np.random.default_rng(spec["seed"] + 1000)
    lin, lout = net.input_layers()[0], net.output_layers()[0]
    rows = spec["hp"] * spec["S"]
    seq = []
    for _ in range(spec["iters"]):
        x = rng.uniform(-1.0, 1.0, size=(rows, lin.size))
        if spec.get("criterion", "cross_entropy_softmax") == "cross_entropy_softmax":
            t = rng.integers(0, lout.size, size=rows)
        else:
            t = rng.uniform(-1.0, 1.0, size=(rows, lout.size))
        seq.append((x, t))
    return seq


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def normwise(a, b) -> float:
    """||a - b||_inf / ||b||_inf (SURVEY.md App. C metric; 0/0 -> 0)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = float(np.abs(b).max()) if b.size else 0.0
    num = float(np.abs(a - b).max()) if b.size else 0.0
    if den == 0.0:
        return num
    return num / den
