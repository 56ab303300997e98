"""ORACLE / CPU-BASELINE INFRASTRUCTURE ONLY.  Never imported by the product path.

Runs the reference implementation itself -- the unmodified ``rnngraph``
package (numba-JIT float64 kernels, /root/reference/pkg/src/rnngraph) --
through its own public ``train_loop`` (engine.py:711-762) to time the CPU
baseline of record on the host cores of whatever box runs it.

The reference is pure Python: ``oracle/build_ref.sh`` installs it (pip,
offline, no deps) into ``oracle/_ref/`` -- git-ignored, but shipped with the
repo snapshot to the GPU box like the built ``.so``, where ``/root/reference``
does not exist.  Only bench.py (its ``--impl reference`` arm and the
``cpu_baseline`` leg) and tools/ call this module.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def load_reference():
    """Import the installed reference (``rnngraph`` from oracle/_ref) with the
    numba pool sized to every host thread (the reference sizes it at import,
    kernels.py:62-75).  Returns the module, or None when it is not installed."""
    if not os.path.isdir(os.path.join(REF_DIR, "rnngraph")):
        return None
    os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count() or 1))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rgb_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import rnngraph

    return rnngraph


def numba_info() -> dict:
    import numba

    return {"numba": numba.__version__, "threads": int(numba.config.NUMBA_NUM_THREADS)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def to_reference(R, net):
    """Our NetworkDef -> the reference's NetworkDef (same ids, by enum value)."""
    layers = tuple(
        R.LayerDef(l.id, l.name, l.size, R.Aggregation(l.aggregation.value), R.Activation(l.activation.value),
                   R.Role(l.role.value))
        for l in net.layers)
    conns = tuple(R.ConnectionDef(c.id, c.src, c.dst, c.delay, R.WeightKind(c.weight_kind.value))
                  for c in net.connections)
    return R.NetworkDef(layers=layers, connections=conns)


class DenseSource:
    """StreamSource (engine.py:670-678): U(-1, 1) dense inputs and uniform class
    targets, the synthetic data of bench.py, produced inside the reference's
    own timed region (train_loop times next_batch too, engine.py:733-734)."""

    def __init__(self, R, n_in: int, n_out: int, n_streams: int, seed: int = 0):
        self.R, self.n_in, self.n_out, self.n_streams = R, n_in, n_out, n_streams
        self.rng = np.random.default_rng(seed)

    def next_batch(self, h_prime: int):
        from types import SimpleNamespace

        rows = h_prime * self.n_streams
        x = self.rng.uniform(-1.0, 1.0, size=(rows, self.n_in))
        return SimpleNamespace(inputs=self.R.Batch(x, h_prime, self.n_streams),
                               targets=self.rng.integers(0, self.n_out, size=rows, dtype=np.int64),
                               new_sequence=None)


def time_train_loop(net, S: int, h: int, hp: int, lr: float, warm: int, iters: int, *, frame_parallel: bool = True,
                    seed: int = 0):
    """Run the reference's train_loop for warm + iters iterations and return
    (frames/s over the timed iterations, timed iteration count, timed seconds,
    per-iteration seconds), from the reference's own per-iteration
    perf_counter (IterationMetrics, engine.py:751-757)."""
    R = load_reference()
    if R is None:
        raise RuntimeError("reference not installed in oracle/_ref (run oracle/build_ref.sh)")
    rnet = to_reference(R, net)
    lin, lout = rnet.input_layers()[0], rnet.output_layers()[0]
    src = DenseSource(R, lin.size, lout.size, S, seed)
    cfg = R.TrainConfig(h=h, h_prime=hp, lr=lr, iterations=warm + iters, seed=seed, frame_parallel=frame_parallel)
    _, metrics = R.train_loop(rnet, src, cfg)
    timed = metrics[warm:]
    secs = sum(m.seconds for m in timed)
    frames = sum(m.frames for m in timed)
    return frames / secs, len(timed), secs, [m.seconds for m in timed]
