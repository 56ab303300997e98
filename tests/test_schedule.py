"""The analyser's device program, interpreted in float64 on the CPU
(tests/program_sim.py), reproduces the oracle's outputs, errors and gradients:
this pins the schedule (hoisting, packing, ring/window addressing) before any
kernel runs."""
from __future__ import annotations

import numpy as np
import pytest

from golden_cases import CASES
from oracle import engine_np as O
from oracle_util import case_inputs, case_net, normwise
from paper_1503_02852_b200 import (build_custom_graph, build_elman, build_lstm, build_stacked_lstm, condense)
from paper_1503_02852_b200.schedule import EngineError, build_program
from program_sim import Sim, flat_weights, unflat


def _check_buckets(net, prog, ctx):
    """Bucketed backward: every dense edge's gradient range is all-reduced
    exactly once, after the dW step that wrote it, and never written again."""
    L = prog.layout
    covered = np.zeros(L.n_params, dtype=int)
    for ranges, written in ctx["ar"]:
        for a, b in ranges:
            covered[a:b] += 1
            for c in net.iter_dense():
                o = L.w_off[c.id]
                n = net.layer(c.dst).size * net.layer(c.src).size
                if a <= o < b:
                    assert (o, o + n) in written, c.id
    for c in net.iter_dense():
        o = L.w_off[c.id]
        n = net.layer(c.dst).size * net.layer(c.src).size
        assert (covered[o:o + n] == 1).all(), c.id
    assert len(ctx["dw_written"]) == len(set(ctx["dw_written"]))


def _run_both(net, S, h, hp, iters, lr, seed, sequential=False, chunk=None, crit=O.CE, hw=None, bucketed=False):
    cg = condense(net)
    prog = build_program(net, cg, S, h, chunk)
    sim = Sim(prog.words)
    W = O.init_weights(net, seed)
    Wsim = {k: v.copy() for k, v in W.items()}
    st = O.History(net, S, h)
    rng = np.random.default_rng(seed + 7)
    lin, lout = net.input_layers()[0], net.output_layers()[0]
    worst = 0.0
    hw = hw or h
    for _ in range(iters):
        x = rng.uniform(-1, 1, size=(hp * S, lin.size))
        if crit == O.CE:
            t = rng.integers(0, lout.size, size=hp * S)
        else:
            t = rng.uniform(-1, 1, size=(hp * S, lout.size))
        out = O.forward_chunk(net, cg, W, st, x)
        w, wt = flat_weights(prog, Wsim)
        out_s = sim.forward(w, x, sequential=sequential)
        worst = max(worst, normwise(out_s, out))
        d = O.inject_output_error(t, out)
        g = O.backward_window(net, cg, W, st, st.cursor, hw, hp, d)
        sim.set_injection(O.inject_output_error(t, out_s))
        gflat = np.zeros(prog.layout.n_params)
        ctx = sim.backward(wt, gflat, hw, hp, sequential=sequential, bucketed=bucketed)
        if bucketed:
            _check_buckets(net, prog, ctx)
        gs = unflat(prog, net, gflat)
        for cid in g:
            worst = max(worst, normwise(gs[cid], g[cid]))
        O.sgd_update(W, g, lr)
        O.sgd_update(Wsim, gs, lr)
    return worst


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("sequential", [False, True])
def test_program_matches_oracle_on_golden_cases(name, sequential):
    spec = CASES[name]
    if spec.get("compact") and sequential:
        pytest.skip("covered by the small cases")
    net = case_net(name)
    worst = _run_both(net, spec["S"], spec["h"], spec["hp"], spec["iters"] + 2, spec["lr"], spec["seed"],
                      sequential=sequential, chunk=spec["hp"],
                      crit=spec.get("criterion", O.CE))
    assert worst < 1e-10


@pytest.mark.parametrize("name", sorted(CASES))
def test_bucketed_backward_matches_oracle(name):
    """The multi-GPU backward (per-supernode dW buckets + all-reduce markers,
    SURVEY §8(e)) computes the same gradients, and every bucket is complete
    when its all-reduce is issued."""
    spec = CASES[name]
    if spec.get("frame_parallel") is False:
        pytest.skip("bucketed only for the hoisted schedule")
    net = case_net(name)
    worst = _run_both(net, spec["S"], spec["h"], spec["hp"], spec["iters"], spec["lr"], spec["seed"],
                      chunk=spec["hp"], crit=spec.get("criterion", O.CE), bucketed=True)
    assert worst < 1e-10


def test_cfg4_buckets_follow_reverse_topological_order():
    net = build_stacked_lstm(1024, [1024] * 3, 1024)
    prog = build_program(net, condense(net), 4, 4, 2)
    buckets = prog.stats["buckets"]
    assert len(buckets) == 4  # one before each SCC loop (top layer first), one at the end
    off = prog.layout.w_off

    def bucket_of(src, dst):
        o = off[net.find_connection(src, dst).id]
        return [i for i, bk in enumerate(buckets) if any(a <= o < b for a, b in bk)]

    assert bucket_of("out_prod_2", "out") == [0]       # the output layer's edges first
    assert bucket_of("cell_2", "in_gate_2") == [1]     # layer 2's SCC before layer 1's loop
    assert bucket_of("in", "in_gate_0") == [3]         # the bottom layer last
    total = sum(b - a for bk in buckets for a, b in bk)
    assert total >= sum(net.layer(c.dst).size * net.layer(c.src).size for c in net.iter_dense())


@pytest.mark.parametrize("S,h,hp", [(1, 5, 2), (3, 7, 3), (2, 4, 4), (2, 9, 1)])
def test_program_chunk_shapes(S, h, hp):
    assert _run_both(build_custom_graph(4, 5, 3), S, h, hp, 6, 0.05, 3) < 1e-10
    assert _run_both(build_stacked_lstm(3, (4, 2), 3), S, h, hp, 5, 0.05, 4, chunk=hp) < 1e-10


def test_shorter_window_than_state():
    assert _run_both(build_lstm(3, 4, 3), 2, 8, 2, 7, 0.05, 5, hw=5) < 1e-10


def test_random_graphs():
    """Random valid graphs with multiplicative layers, identity edges, width-1
    layers and multi-frame delays."""
    from paper_1503_02852_b200.netdef import (Activation, Aggregation, ConnectionDef, LayerDef, NetworkDef, Role,
                                              WeightKind, validate)
    rng = np.random.default_rng(123)
    done = 0
    while done < 25:
        n_hidden = int(rng.integers(1, 6))
        width = int(rng.integers(2, 5))
        layers = [LayerDef(0, "in", 3, role=Role.INPUT), LayerDef(1, "bias", 1)]
        for i in range(n_hidden):
            mul = rng.random() < 0.3
            act = Activation.IDENTITY if mul else [Activation.TANH, Activation.SIGMOID, Activation.IDENTITY][
                int(rng.integers(3))]
            layers.append(LayerDef(2 + i, f"h{i}", width if rng.random() < 0.8 else 1,
                                   Aggregation.MULTIPLICATIVE if mul else Aggregation.ADDITIVE, act))
        layers.append(LayerDef(len(layers), "out", 3, activation=Activation.SOFTMAX, role=Role.OUTPUT))
        conns = []
        hid = list(range(2, 2 + n_hidden))
        for h_ in hid:
            conns.append((0, h_, 0, WeightKind.DENSE))
        for _ in range(int(rng.integers(2, 8))):
            a, b = int(rng.choice(hid + [1])), int(rng.choice(hid))
            d = int(rng.integers(0, 3))
            kind = WeightKind.IDENTITY if (layers[a].size == layers[b].size and rng.random() < 0.4) else WeightKind.DENSE
            conns.append((a, b, d, kind))
        conns.append((int(rng.choice(hid)), len(layers) - 1, 0, WeightKind.DENSE))
        conns.append((1, len(layers) - 1, 0, WeightKind.DENSE))
        net = NetworkDef(tuple(layers), tuple(ConnectionDef(i, a, b, d, k) for i, (a, b, d, k) in enumerate(conns)))
        if not validate(net).ok or any(
                len(net.anterior(l.id)) > 4 for l in net.layers if l.aggregation is Aggregation.MULTIPLICATIVE):
            continue
        if any(net.posterior(l.id) for l in net.layers if l.activation is Activation.SOFTMAX):
            continue
        for seq in (False, True):
            assert _run_both(net, 2, 6, 3, 4, 0.05, done, sequential=seq) < 1e-9, (conns, seq)
        done += 1


def test_engine_rejects_two_inputs():
    from paper_1503_02852_b200.netdef import ConnectionDef, LayerDef, NetworkDef, Role
    net = NetworkDef(
        layers=(LayerDef(0, "a", 1, role=Role.INPUT), LayerDef(1, "b", 1, role=Role.INPUT),
                LayerDef(2, "out", 1, role=Role.OUTPUT)),
        connections=(ConnectionDef(0, 0, 2), ConnectionDef(1, 1, 2)),
    )
    with pytest.raises(EngineError, match="exactly one input"):
        build_program(net, condense(net), 1, 2)


def test_lstm_launch_counts():
    """One launch per backward frame, two per forward frame."""
    net = build_lstm(39, 128, 39)
    p = build_program(net, condense(net), 1, 32, 16)
    assert p.stats["backward"]["loop_launches_per_frame"] == 1
    assert p.stats["forward"]["loop_launches_per_frame"] == 2
    e = build_elman(3, 4, 5)
    assert build_program(e, condense(e), 1, 4).stats["backward"]["loop_launches_per_frame"] == 1
