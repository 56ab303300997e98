"""Reference topologies as plain graph structure.

``build_elman`` and ``build_lstm`` reproduce the layer and connection order of
the reference builders (``/root/reference/pkg/src/rnngraph/builders.py:58-149``)
exactly, because connection ids key the weight/gradient stores and the
parity fixtures.  ``build_stacked_lstm`` (configs 2-4 of BASELINE.json) and
``build_custom_graph`` (config 5) are new: the reference has no stacked
builder; they use the same per-block wiring, and the one-block
stacked network is identical to ``build_lstm``.
"""

from __future__ import annotations

from typing import Sequence

from .netdef import (
    Activation,
    Aggregation,
    ConnectionDef,
    LayerDef,
    NetworkDef,
    Role,
    WeightKind,
    validate,
)

__all__ = ["build_elman", "build_lstm", "build_stacked_lstm", "build_custom_graph", "count_params"]

_ID = WeightKind.IDENTITY


class _Net:
    """Tiny mutable accumulator that hands out ids in insertion order."""

    def __init__(self):
        self._layers: list[LayerDef] = []
        self._conns: list[ConnectionDef] = []
        self._ids: dict[str, int] = {}

    def add(self, name, size, *, mul=False, act=Activation.IDENTITY, role=Role.HIDDEN):
        lid = len(self._layers)
        agg = Aggregation.MULTIPLICATIVE if mul else Aggregation.ADDITIVE
        self._layers.append(LayerDef(lid, name, size, agg, act, role))
        self._ids[name] = lid

    def edge(self, src, dst, delay=0, kind=WeightKind.DENSE):
        cid = len(self._conns)
        self._conns.append(ConnectionDef(cid, self._ids[src], self._ids[dst], delay, kind))

    def finish(self) -> NetworkDef:
        net = NetworkDef(layers=tuple(self._layers), connections=tuple(self._conns))
        validate(net).raise_if_failed()
        return net


def build_elman(n_in, n_hidden, n_out, *, include_bias=True,
                hidden_activation=Activation.TANH, output_activation=Activation.SOFTMAX):
    """h(t) = f(W_xh x(t) + W_hh h(t-1) + b); out = g(W_hy h + b)."""
    g = _Net()
    g.add("in", n_in, role=Role.INPUT)
    if include_bias:
        g.add("bias", 1)
    g.add("hidden", n_hidden, act=hidden_activation)
    g.add("out", n_out, act=output_activation, role=Role.OUTPUT)
    g.edge("in", "hidden")
    g.edge("hidden", "hidden", 1)
    g.edge("hidden", "out")
    if include_bias:
        g.edge("bias", "hidden")
        g.edge("bias", "out")
    return g.finish()


def _lstm_block(g: _Net, n: int, sfx: str, *, forget_gate: bool):
    """Layers of one peephole-LSTM block; returns the name mangler."""
    L = lambda base: base + sfx  # noqa: E731
    g.add(L("cell_in"), n, act=Activation.TANH)
    g.add(L("in_gate"), n, act=Activation.SIGMOID)
    if forget_gate:
        g.add(L("forget_gate"), n, act=Activation.SIGMOID)
    g.add(L("in_prod"), n, mul=True)
    if forget_gate:
        g.add(L("forget_prod"), n, mul=True)
    g.add(L("cell"), n)
    g.add(L("cell_act"), n, act=Activation.TANH)
    g.add(L("out_gate"), n, act=Activation.SIGMOID)
    g.add(L("out_prod"), n, mul=True)
    return L


def _lstm_edges(g: _Net, src: str, L, *, peepholes, forget_gate, include_bias,
                output_peephole_delay, bias_out: bool):
    gates = [L("cell_in"), L("in_gate"), L("out_gate")] + ([L("forget_gate")] if forget_gate else [])
    for gate in gates:
        g.edge(src, gate)
    if include_bias:
        for gate in gates:
            g.edge("bias", gate)
        if bias_out:
            g.edge("bias", "out")
    if peepholes:
        g.edge(L("cell"), L("in_gate"), 1)
        if forget_gate:
            g.edge(L("cell"), L("forget_gate"), 1)
        g.edge(L("cell"), L("out_gate"), output_peephole_delay)
    g.edge(L("cell_in"), L("in_prod"), kind=_ID)
    g.edge(L("in_gate"), L("in_prod"), kind=_ID)
    if forget_gate:
        g.edge(L("cell"), L("forget_prod"), 1, _ID)
        g.edge(L("forget_gate"), L("forget_prod"), kind=_ID)
        g.edge(L("forget_prod"), L("cell"), kind=_ID)
    else:
        g.edge(L("cell"), L("cell"), 1, _ID)
    g.edge(L("in_prod"), L("cell"), kind=_ID)
    g.edge(L("cell"), L("cell_act"), kind=_ID)
    g.edge(L("cell_act"), L("out_prod"), kind=_ID)
    g.edge(L("out_gate"), L("out_prod"), kind=_ID)


def build_stacked_lstm(n_in: int, cells: Sequence[int], n_out: int, *, peepholes=True,
                       forget_gate=True, include_bias=True, output_peephole_delay=0,
                       output_activation=Activation.SOFTMAX) -> NetworkDef:
    """``len(cells)`` peephole-LSTM blocks in series: block b's gates read
    block b-1's ``out_prod`` (block 0 reads ``in``); the last block's
    ``out_prod`` feeds ``out``.  Layer names carry a ``_b`` suffix when there is
    more than one block.  One block reproduces ``build_lstm`` id for id."""
    if output_peephole_delay not in (0, 1):
        raise ValueError(f"output_peephole_delay must be 0 or 1, got {output_peephole_delay}")
    if not cells:
        raise ValueError("need at least one LSTM block")
    opts = dict(peepholes=peepholes, forget_gate=forget_gate, include_bias=include_bias,
                output_peephole_delay=output_peephole_delay)
    g = _Net()
    g.add("in", n_in, role=Role.INPUT)
    if include_bias:
        g.add("bias", 1)
    suffixes = [""] if len(cells) == 1 else [f"_{b}" for b in range(len(cells))]
    namers = [_lstm_block(g, n, s, forget_gate=forget_gate) for n, s in zip(cells, suffixes)]
    g.add("out", n_out, act=output_activation, role=Role.OUTPUT)
    src = "in"
    for b, L in enumerate(namers):
        _lstm_edges(g, src, L, bias_out=(b == 0), **opts)
        src = L("out_prod")
    g.edge(src, "out")
    return g.finish()


def build_lstm(n_in, n_cells, n_out, *, peepholes=True, forget_gate=True, include_bias=True,
               output_peephole_delay=0, output_activation=Activation.SOFTMAX) -> NetworkDef:
    """Peephole LSTM (forget gate, full-matrix peepholes, bias layer), same
    ids as the reference ``build_lstm`` (builders.py:83-149)."""
    return build_stacked_lstm(
        n_in, [n_cells], n_out, peepholes=peepholes, forget_gate=forget_gate,
        include_bias=include_bias, output_peephole_delay=output_peephole_delay,
        output_activation=output_activation,
    )


def build_custom_graph(n_in: int = 39, n_hidden: int = 128, n_out: int = 39) -> NetworkDef:
    """Config 5: a generalized graph RNN with
    multiplicative layers and delay-1/delay-2 edges, no peepholes.

    SCCs: {a, g, m, r} (dense zero-delay m->r inside, so two grid barriers per
    frame) and {v, w}; u is a simple node between them.
    """
    g = _Net()
    T, S = Activation.TANH, Activation.SIGMOID
    g.add("in", n_in, role=Role.INPUT)
    g.add("bias", 1)
    g.add("a", n_hidden, act=T)
    g.add("g", n_hidden, act=S)
    g.add("m", n_hidden, mul=True)
    g.add("r", n_hidden, act=T)
    g.add("u", n_hidden, act=S)
    g.add("v", n_hidden, mul=True)
    g.add("w", n_hidden, act=T)
    g.add("out", n_out, act=Activation.SOFTMAX, role=Role.OUTPUT)
    for dst in ("a", "g", "u"):
        g.edge("in", dst)
    for dst in ("a", "g", "u", "w", "out"):
        g.edge("bias", dst)
    g.edge("r", "a", 2)
    g.edge("m", "g", 1)
    g.edge("a", "m", kind=_ID)
    g.edge("g", "m", kind=_ID)
    g.edge("m", "r")
    g.edge("r", "r", 1)
    g.edge("r", "u")
    g.edge("u", "v", kind=_ID)
    g.edge("w", "v", 1, _ID)
    g.edge("v", "w")
    g.edge("w", "out")
    g.edge("m", "out")
    return g.finish()


def count_params(net: NetworkDef) -> int:
    """Trainable scalars (dense matrices only)."""
    return sum(net.layer(c.dst).size * net.layer(c.src).size for c in net.iter_dense())
