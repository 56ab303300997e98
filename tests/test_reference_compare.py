"""The dependency analyser against the reference itself, on random graphs
(CPU suite; skipped where /root/reference is absent, e.g. on the GPU box).

For 2000 random networks -- valid and invalid: multiplicative layers, identity
edges of matching and mismatching widths, width-1 layers, delays 0..2 and so
zero-delay cycles, duplicate edges, extra input / output layers -- our
``validate`` must report the same rule set as the reference's
(``netdef.py:282-405``), and on the valid ones ``tarjan_scc`` / ``condense``
(``condense.py:50-198``) must return the same components, recurrent flags,
internal orders, crossing edges, topological order and frontier levels, and
``schedule_text`` the same text."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1503_02852_b200 import condense, schedule_text, tarjan_scc, validate
from paper_1503_02852_b200.netdef import (Activation, Aggregation, ConnectionDef, LayerDef, NetworkDef, Role,
                                          WeightKind)

N_GRAPHS = 2000


def _random_net(rng):
    return _careful_net(rng) if rng.random() < 0.5 else _wild_net(rng)


def _careful_net(rng):
    """Mostly-valid graphs: one input / output, back edges delayed, identity
    edges between equal widths, multiplicative layers with identity output."""
    n_hidden = int(rng.integers(1, 8))
    layers = [LayerDef(0, "in", 3, role=Role.INPUT), LayerDef(1, "bias", 1)]
    for i in range(n_hidden):
        mul = rng.random() < 0.3
        act = Activation.IDENTITY if mul else [Activation.TANH, Activation.SIGMOID, Activation.IDENTITY][
            int(rng.integers(3))]
        layers.append(LayerDef(2 + i, f"h{i}", int(rng.choice([1, 2, 2, 3])),
                               Aggregation.MULTIPLICATIVE if mul else Aggregation.ADDITIVE, act))
    out = len(layers)
    layers.append(LayerDef(out, "out", 3, activation=Activation.SOFTMAX, role=Role.OUTPUT))
    hid = list(range(2, 2 + n_hidden))
    conns = [(0, h, 0, WeightKind.DENSE) for h in hid if rng.random() < 0.8]
    for _ in range(int(rng.integers(1, 10))):
        a, b = int(rng.choice(hid + [1, 0])), int(rng.choice(hid))
        d = int(rng.integers(1, 3)) if a >= b else int(rng.integers(0, 3))
        same = layers[a].size == layers[b].size and a != 0
        kind = WeightKind.IDENTITY if same and rng.random() < 0.4 else WeightKind.DENSE
        conns.append((a, b, d, kind))
    conns.append((int(rng.choice(hid)), out, 0, WeightKind.DENSE))
    if rng.random() < 0.7:
        conns.append((1, out, 0, WeightKind.DENSE))
    order = rng.permutation(len(conns))
    return NetworkDef(tuple(layers), tuple(ConnectionDef(i, *conns[j]) for i, j in enumerate(order)))


def _wild_net(rng):
    n_hidden = int(rng.integers(1, 7))
    layers = [LayerDef(0, "in", int(rng.integers(1, 4)), role=Role.INPUT), LayerDef(1, "bias", 1)]
    for i in range(n_hidden):
        mul = rng.random() < 0.3
        act = [Activation.TANH, Activation.SIGMOID, Activation.IDENTITY, Activation.SOFTMAX][int(rng.integers(4))]
        if mul and rng.random() < 0.8:
            act = Activation.IDENTITY
        layers.append(LayerDef(2 + i, f"h{i}", int(rng.choice([1, 2, 3])),
                               Aggregation.MULTIPLICATIVE if mul else Aggregation.ADDITIVE, act))
    n_out = 2 if rng.random() < 0.05 else 1
    for k in range(n_out):
        layers.append(LayerDef(len(layers), f"out{k}", 3, activation=Activation.SOFTMAX, role=Role.OUTPUT))
    if rng.random() < 0.05:
        layers.append(LayerDef(len(layers), "in2", 2, role=Role.INPUT))
    ids = list(range(len(layers)))
    conns = []
    for _ in range(int(rng.integers(2, 12))):
        a, b = int(rng.choice(ids)), int(rng.choice(ids))
        d = int(rng.choice([0, 0, 1, 2]))
        kind = WeightKind.IDENTITY if rng.random() < 0.25 else WeightKind.DENSE
        conns.append((a, b, d, kind))
    for h in range(2, 2 + n_hidden):
        if rng.random() < 0.7:
            conns.append((0, h, 0, WeightKind.DENSE))
    conns.append((int(rng.integers(2, 2 + n_hidden)), 2 + n_hidden, 0, WeightKind.DENSE))
    order = rng.permutation(len(conns))
    return NetworkDef(tuple(layers), tuple(ConnectionDef(i, *conns[j]) for i, j in enumerate(order)))


def _ref_net(R, net):
    layers = tuple(R.LayerDef(l.id, l.name, l.size, R.Aggregation(l.aggregation.value),
                              R.Activation(l.activation.value), R.Role(l.role.value)) for l in net.layers)
    conns = tuple(R.ConnectionDef(c.id, c.src, c.dst, c.delay, R.WeightKind(c.weight_kind.value))
                  for c in net.connections)
    return R.NetworkDef(layers=layers, connections=conns)


def _cg_tuple(cg):
    return ([(n.members, n.recurrent, n.internal_order) for n in cg.nodes], tuple(cg.edges), tuple(cg.topo_order),
            tuple(tuple(lv) for lv in cg.frontier_levels), dict(cg.node_of_layer))


def test_validate_and_condense_match_the_reference(reference):
    R = reference
    import importlib
    RC = importlib.import_module("rnngraph.condense")
    rng = np.random.default_rng(2024)
    n_valid = 0
    for i in range(N_GRAPHS):
        net = _random_net(rng)
        rnet = _ref_net(R, net)
        ours = sorted({v.rule for v in validate(net).violations})
        ref = sorted({v.rule for v in R.validate(rnet).violations})
        assert ours == ref, (i, ours, ref)
        if ref:
            continue
        n_valid += 1
        assert [tuple(c) for c in tarjan_scc(net)] == [tuple(c) for c in R.tarjan_scc(rnet)], i
        assert _cg_tuple(condense(net)) == _cg_tuple(R.condense(rnet)), i
        assert schedule_text(condense(net), net) == RC.schedule_text(R.condense(rnet), rnet), i
    assert n_valid >= 300, n_valid  # enough valid graphs exercise the condensation


def test_cfg_graphs_match_the_reference(reference):
    """The benchmarked graphs: stacked LSTMs (cfg2-4) and the custom graph (cfg5)."""
    from paper_1503_02852_b200 import build_custom_graph, build_lstm, build_stacked_lstm
    R = reference
    for net in (build_lstm(39, 128, 39), build_stacked_lstm(1024, [1024] * 3, 1024), build_custom_graph()):
        rnet = _ref_net(R, net)
        assert R.validate(rnet).ok and validate(net).ok
        assert _cg_tuple(condense(net)) == _cg_tuple(R.condense(rnet))
