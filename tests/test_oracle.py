"""The oracle (oracle/engine_np.py) is pinned against the reference's own outputs
(golden fixtures made by tests/golden/make_golden.py) and the reference's
known-answer tests."""
from __future__ import annotations

import math

import numpy as np
import pytest

from golden_cases import CASES
from oracle import engine_np as O
from oracle_util import case_inputs, case_net, load_golden, normwise
from paper_1503_02852_b200 import build_elman, build_lstm, condense
from paper_1503_02852_b200.netdef import ConnectionDef, LayerDef, NetworkDef, Role, WeightKind


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_golden(name):
    spec = CASES[name]
    gold = load_golden(name)
    net = case_net(name)
    cg = condense(net)
    W = O.init_weights(net, spec["seed"])
    tol = 2e-6 if spec.get("compact") else 1e-11
    if not spec.get("compact"):
        for cid, w in W.items():
            assert np.array_equal(w, gold[f"w0_{cid}"]), cid  # same PCG64 draw sequence
    st = O.History(net, spec["S"], spec["h"])
    crit = spec.get("criterion", O.CE)
    fp = spec.get("frame_parallel", True)
    cap = {}
    for it, (x, t) in enumerate(case_inputs(name, net)):
        out = O.forward_chunk(net, cg, W, st, x, frame_parallel=fp)
        assert normwise(out, gold[f"out_{it}"]) < tol
        loss = O.loss_value(t, out, crit)
        assert abs(loss - float(gold[f"loss_{it}"])) <= tol * max(1.0, abs(loss))
        d = O.inject_output_error(t, out)
        g = O.backward_window(net, cg, W, st, st.cursor, spec["h"], spec["hp"], d,
                              frame_parallel=fp, capture=cap)
        for cid in g:
            assert normwise(g[cid], gold[f"g_{it}_{cid}"]) < tol, (it, cid)
        O.sgd_update(W, g, spec["lr"])
    for lid, v in cap["delta"].items():
        assert normwise(v, gold[f"delta_{lid}"]) < tol, ("delta", lid)
    for cid, v in cap["eps"].items():
        assert normwise(v, gold[f"eps_{cid}"]) < tol, ("eps", cid)
    if not spec.get("compact"):
        for cid, w in W.items():
            assert normwise(w, gold[f"w_final_{cid}"]) < tol


def test_cumsum_known_answer():
    """reference tests/test_engine.py:84-92: out(t) = in(t) + out(t-1) -> [1, 3, 6]."""
    net = NetworkDef(
        layers=(LayerDef(0, "in", 1, role=Role.INPUT), LayerDef(1, "out", 1, role=Role.OUTPUT)),
        connections=(ConnectionDef(0, 0, 1, weight_kind=WeightKind.IDENTITY),
                     ConnectionDef(1, 1, 1, delay=1, weight_kind=WeightKind.IDENTITY)),
    )
    st = O.History(net, 1, 3)
    out = O.forward_chunk(net, condense(net), {}, st, np.array([[1.0], [2.0], [3.0]]))
    assert np.array_equal(out, [[1.0], [3.0], [6.0]])


def test_loss_known_answers():
    """reference tests/test_engine.py:215-223."""
    onehot = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert O.loss_value(np.array([1, 0]), onehot) == 0.0
    uniform = np.full((3, 4), 0.25)
    assert abs(O.loss_value(np.array([0, 1, 2]), uniform) - 3 * math.log(4)) < 1e-12
    assert O.loss_value(np.array([[0.0, 4.0]]), np.array([[1.0, 2.0]]), O.MSE) == 2.5


def test_multi_stream_equals_sum_of_single_streams():
    """reference tests/test_acceptance.py:180-207 (restated with tolerance)."""
    net = build_elman(5, 4, 5)
    cg = condense(net)
    rng = np.random.default_rng(11)
    S, hp, h = 4, 3, 6
    xs = rng.uniform(-1, 1, size=(3, S, hp, 5))
    ts = rng.integers(0, 5, size=(3, S, hp))
    W = O.init_weights(net, 9)

    def run(streams):
        st = O.History(net, len(streams), h)
        g = None
        for c in range(3):
            x = np.stack([xs[c, s] for s in streams], axis=1).reshape(-1, 5)
            t = np.stack([ts[c, s] for s in streams], axis=1).reshape(-1)
            out = O.forward_chunk(net, cg, W, st, x)
            g = O.backward_window(net, cg, W, st, st.cursor, h, hp, O.inject_output_error(t, out))
        return g

    multi = run([0, 1, 2, 3])
    single = [run([s]) for s in range(4)]
    for cid in multi:
        assert normwise(multi[cid], sum(g[cid] for g in single)) < 1e-12


def test_lstm_forward_matches_hand_recurrence():
    """reference tests/oracles.py:122-173 + test_acceptance.py:100-126."""
    net = build_lstm(3, 4, 3)
    W = O.init_weights(net, 1)
    xs = np.random.default_rng(18).uniform(-1, 1, size=(50, 3))
    st = O.History(net, 1, 50)
    out = O.forward_chunk(net, condense(net), W, st, xs)
    Wn = lambda s, d: W[net.find_connection(s, d).id]  # noqa: E731
    sig = lambda v: 1 / (1 + np.exp(-v))  # noqa: E731
    c_prev = np.zeros(4)
    for t, x in enumerate(xs):
        b = lambda d: Wn("bias", d)[:, 0]  # noqa: E731
        g = np.tanh(Wn("in", "cell_in") @ x + b("cell_in"))
        i = sig(Wn("in", "in_gate") @ x + b("in_gate") + Wn("cell", "in_gate") @ c_prev)
        f = sig(Wn("in", "forget_gate") @ x + b("forget_gate") + Wn("cell", "forget_gate") @ c_prev)
        c = c_prev * f + g * i
        o = sig(Wn("in", "out_gate") @ x + b("out_gate") + Wn("cell", "out_gate") @ c)
        z = Wn("out_prod", "out") @ (np.tanh(c) * o) + b("out")
        y = np.exp(z - z.max()) / np.exp(z - z.max()).sum()
        assert np.abs(out[t] - y).max() < 1e-10
        c_prev = c
