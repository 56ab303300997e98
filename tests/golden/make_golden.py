"""Generate the golden fixtures that pin the oracle (run in the build container).

Imports the reference package read-only from /root/reference/pkg/src and
drives its public API (``Weights.init``, ``StreamState``, ``forward_chunk``,
``loss_value``, ``inject_output_error``, ``backward_window``, ``sgd_update``;
engine.py:126-612) over a few small networks and config 1, recording per
iteration the outputs, loss and loss gradient, plus every delta and eps of
the last window.  delta/eps are locals of ``backward_window``; they are read
by wrapping ``GradStore.zeros`` (called at engine.py:580, after all errors are
final) and inspecting the caller's frame -- the reference is not modified.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Writes tests/golden/<case>.npz.  The GPU box never runs this file.
"""

from __future__ import annotations

import inspect
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import rnngraph as R  # noqa: E402
from rnngraph import engine as RE  # noqa: E402

from paper_1503_02852_b200 import builders as B  # noqa: E402

from golden_cases import CASES  # noqa: E402  (tests/golden/golden_cases.py)


def to_reference(net):
    """Our NetworkDef -> reference NetworkDef (by enum value)."""
    layers = tuple(
        R.LayerDef(l.id, l.name, l.size, R.Aggregation(l.aggregation.value),
                   R.Activation(l.activation.value), R.Role(l.role.value))
        for l in net.layers)
    conns = tuple(R.ConnectionDef(c.id, c.src, c.dst, c.delay, R.WeightKind(c.weight_kind.value))
                  for c in net.connections)
    return R.NetworkDef(layers=layers, connections=conns)


_captured: dict = {}
_orig_zeros = RE.GradStore.zeros.__func__


def _spy_zeros(cls, net):
    frame = inspect.currentframe().f_back
    loc = frame.f_locals
    if "delta" in loc and "eps" in loc:
        _captured["delta"] = {k: v.copy() for k, v in loc["delta"].items()}
        _captured["eps"] = {k: v.copy() for k, v in loc["eps"].items()}
    return _orig_zeros(cls, net)


def run_case(name: str, spec: dict) -> dict:
    ours = getattr(B, spec["builder"])(*spec["args"], **spec.get("kwargs", {}))
    net = to_reference(ours)
    cg = R.condense(net)
    S, h, hp, iters = spec["S"], spec["h"], spec["hp"], spec["iters"]
    lr, seed = spec["lr"], spec["seed"]
    crit = R.Criterion(spec.get("criterion", "cross_entropy_softmax"))
    fp = spec.get("frame_parallel", True)
    w = R.Weights.init(net, seed)
    state = R.StreamState(net, S, h)
    rng = np.random.default_rng(seed + 1000)
    lin, lout = net.input_layers()[0], net.output_layers()[0]
    rec: dict[str, np.ndarray] = {}
    for c in sorted(w.w):
        rec[f"w0_{c}"] = w.w[c].copy()
    RE.GradStore.zeros = classmethod(_spy_zeros)
    try:
        for it in range(iters):
            x = rng.uniform(-1.0, 1.0, size=(hp * S, lin.size))
            if crit is R.Criterion.CROSS_ENTROPY_SOFTMAX:
                tgt = rng.integers(0, lout.size, size=hp * S)
            else:
                tgt = rng.uniform(-1.0, 1.0, size=(hp * S, lout.size))
            out = R.forward_chunk(net, cg, w, state, R.Batch(x, hp, S), frame_parallel=fp)
            t_obj = tgt if tgt.ndim == 1 else R.Batch(tgt, hp, S)
            loss = R.loss_value(t_obj, out, crit)
            d = R.inject_output_error(t_obj, out, crit, lout.activation)
            win = R.BpttWindow(t1=state.cursor, h=h, h_prime=hp)
            g = R.backward_window(net, cg, w, state, win, d, frame_parallel=fp)
            rec[f"x_{it}"] = x
            rec[f"tgt_{it}"] = tgt
            rec[f"out_{it}"] = out.values.copy()
            rec[f"loss_{it}"] = np.array(loss)
            for c in sorted(g.g):
                rec[f"g_{it}_{c}"] = g.g[c].copy()
            R.sgd_update(w, g, lr)
    finally:
        RE.GradStore.zeros = classmethod(_orig_zeros)
    for k, v in _captured["delta"].items():
        rec[f"delta_{k}"] = v
    for k, v in _captured["eps"].items():
        rec[f"eps_{k}"] = v
    for c in sorted(w.w):
        rec[f"w_final_{c}"] = w.w[c].copy()
    return rec


def main() -> None:
    for name, spec in CASES.items():
        rec = run_case(name, spec)
        if spec.get("compact"):  # large case: float32 payload, weights regenerated from the seed
            rec = {k: (v.astype(np.float32) if v.dtype == np.float64 and v.ndim else v)
                   for k, v in rec.items() if not k.startswith(("w0_", "w_final_"))}
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **rec)
        print(f"{name}: {len(rec)} arrays, {os.path.getsize(path) / 1024:.0f} KiB")


if __name__ == "__main__":
    sys.path.insert(0, HERE)
    main()
