"""RNNG v1 checkpoints (reference engine.py:615-665): byte-compatible with the
reference in both directions, guards raise CheckpointError."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1503_02852_b200 as P
from paper_1503_02852_b200.engine import read_checkpoint


class _HostWeights:
    """Stand-in exposing Weights.numpy() without a device."""

    def __init__(self, mats):
        self.mats = mats

    def numpy(self):
        return self.mats


def _random_mats(net, seed):
    rng = np.random.default_rng(seed)
    return {c.id: rng.standard_normal((net.layer(c.dst).size, net.layer(c.src).size))
            for c in net.iter_dense()}


@pytest.mark.parametrize("net_fn", [lambda: P.build_lstm(7, 9, 5), lambda: P.build_custom_graph(),
                                    lambda: P.build_stacked_lstm(6, [8, 7], 5)])
def test_roundtrip(tmp_path, net_fn):
    net = net_fn()
    mats = _random_mats(net, 1)
    path = str(tmp_path / "w.rnng")
    P.save_checkpoint(path, net, _HostWeights(mats))
    back = read_checkpoint(path, net)
    assert set(back) == set(mats)
    for cid in mats:
        assert np.array_equal(back[cid], mats[cid])


def test_guards(tmp_path):
    net = P.build_lstm(7, 9, 5)
    path = str(tmp_path / "w.rnng")
    P.save_checkpoint(path, net, _HostWeights(_random_mats(net, 2)))
    with pytest.raises(P.CheckpointError, match="different network"):
        read_checkpoint(path, P.build_lstm(7, 10, 5))
    blob = open(path, "rb").read()
    open(path, "wb").write(blob[:-3])
    with pytest.raises(P.CheckpointError, match="truncated"):
        read_checkpoint(path, net)
    open(path, "wb").write(b"XXXX" + blob[4:])
    with pytest.raises(P.CheckpointError, match="not a checkpoint"):
        read_checkpoint(path, net)


def test_byte_compatible_with_reference(tmp_path, reference):
    """Files written here load in the reference and vice versa (same canonical
    document, hence the same structure hash)."""
    for net in [P.build_lstm(7, 9, 5), P.build_custom_graph()]:
        ref_net = reference.load_network(P.save_network(net))
        assert reference.save_network(ref_net) == P.save_network(net)
        from rnngraph.engine import structure_hash as ref_hash
        assert ref_hash(ref_net) == P.structure_hash(net)
        mats = _random_mats(net, 3)
        ours = str(tmp_path / "ours.rnng")
        P.save_checkpoint(ours, net, _HostWeights(mats))
        from rnngraph.engine import load_checkpoint as ref_load, save_checkpoint as ref_save
        rw = ref_load(ours, ref_net)
        for cid in mats:
            assert np.array_equal(rw.w[cid], mats[cid])
        theirs = str(tmp_path / "theirs.rnng")
        ref_save(theirs, ref_net, reference.Weights.init(ref_net, 11))
        assert open(theirs, "rb").read()[:16] == open(ours, "rb").read()[:16]
        back = read_checkpoint(theirs, net)
        ref_w = reference.Weights.init(ref_net, 11)
        for cid in back:
            assert np.array_equal(back[cid], ref_w.w[cid])
