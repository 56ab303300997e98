"""Device-fed token tapes: the host planner reproduces the reference's
StreamSet token order (dealing, look-ahead targets across document and epoch
boundaries, per-tape reshuffles, new-sequence flags); the device gather
matches the planner."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1503_02852_b200.tapes import TapePlanner


def _corpus(seed, n_docs, max_len):
    rng = np.random.default_rng(seed)
    return [rng.integers(0, 50, size=int(rng.integers(1, max_len))) for _ in range(n_docs)]


def _host_chunk(planner, k):
    pos, new_seq = planner.next_positions(k)
    tok = planner.corpus[pos]
    n = planner.n_streams
    inputs = np.empty(k * n, dtype=np.int64)
    targets = np.empty(k * n, dtype=np.int64)
    for s in range(n):
        inputs[s::n] = tok[s, :k]
        targets[s::n] = tok[s, 1:]
    return inputs, targets, new_seq


@pytest.mark.parametrize("n_docs,max_len,n_streams,k", [(9, 7, 3, 4), (2, 40, 5, 6), (30, 3, 4, 5), (1, 100, 1, 16)])
def test_planner_matches_reference_streams(reference, n_docs, max_len, n_streams, k):
    from rnngraph.data import make_streams
    docs = _corpus(n_docs * 7 + max_len, n_docs, max_len)
    ref = make_streams(docs, n_streams, seed=3)
    ours = TapePlanner(docs, n_streams, seed=3)
    for _ in range(25):  # several epochs of the short tapes
        r = ref.next_batch(k)
        i, t, b = _host_chunk(ours, k)
        assert np.array_equal(r.inputs, i)
        assert np.array_equal(r.targets, t)
        assert np.array_equal(r.new_sequence, b)


def test_planner_guards():
    with pytest.raises(ValueError):
        TapePlanner([], 2, 0)
    with pytest.raises(ValueError):
        TapePlanner([np.array([1, 2])], 5, 0)
