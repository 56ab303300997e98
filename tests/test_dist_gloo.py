"""Multi-rank logic of the stream-sharded data parallelism (dist.py), run on
CPU with the gloo backend at world size 2: each rank computes the loss
gradient of its own stream shard (the oracle stands in for the GPU step),
the flat gradients (weight_offsets layout, as on the device) are summed with
GradientExchange, and the result must equal the single-process gradient over
all streams (reference tests/test_acceptance.py:180-207); after the identical
SGD step the replicas hold identical weights."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1503_02852_b200 import build_lstm, condense
from paper_1503_02852_b200.dist import GradientExchange, shard_streams
from paper_1503_02852_b200.schedule import weight_offsets

S_TOTAL, H, HP, ITERS = 6, 6, 3, 3


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _flatten(net, g):
    off, n = weight_offsets(net)
    flat = np.zeros(max(n, 4))
    for cid, m in g.items():
        flat[off[cid]:off[cid] + m.size] = m.ravel()
    return flat


def _data(net):
    rng = np.random.default_rng(7)
    xs = rng.uniform(-1, 1, size=(ITERS, HP, S_TOTAL, net.input_layers()[0].size))
    ts = rng.integers(0, net.output_layers()[0].size, size=(ITERS, HP, S_TOTAL))
    return xs, ts


def _reference_run(net):
    """Single process, all streams: flat gradient of every iteration."""
    from oracle import engine_np as O
    cg = condense(net)
    W = O.init_weights(net, 1)
    st = O.History(net, S_TOTAL, H)
    xs, ts = _data(net)
    flats = []
    for it in range(ITERS):
        x = xs[it].reshape(HP * S_TOTAL, -1)
        out = O.forward_chunk(net, cg, W, st, x)
        g = O.backward_window(net, cg, W, st, st.cursor, H, HP, O.inject_output_error(ts[it].reshape(-1), out))
        flats.append(_flatten(net, g))
        O.sgd_update(W, g, 0.05)
    return flats, _flatten(net, W)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import engine_np as O
        net = build_lstm(4, 5, 3)
        cg = condense(net)
        lo, hi = shard_streams(S_TOTAL, world, rank)
        W = O.init_weights(net, 1)
        st = O.History(net, hi - lo, H)
        xs, ts = _data(net)
        ex = GradientExchange()
        flats = []
        for it in range(ITERS):
            x = xs[it][:, lo:hi].reshape(HP * (hi - lo), -1)
            out = O.forward_chunk(net, cg, W, st, x)
            g = O.backward_window(net, cg, W, st, st.cursor, H, HP,
                                  O.inject_output_error(ts[it][:, lo:hi].reshape(-1), out))
            flat = torch.from_numpy(_flatten(net, g))
            ex.allreduce_(flat)  # the one exchange step per iteration
            summed = flat.numpy()
            flats.append(summed)
            off, _ = weight_offsets(net)
            for cid in W:  # identical SGD on every rank from the summed gradient
                W[cid] -= 0.05 * summed[off[cid]:off[cid] + W[cid].size].reshape(W[cid].shape)
        q.put((rank, flats, _flatten(net, W)))
    finally:
        dist.destroy_process_group()


def test_shard_streams():
    assert shard_streams(512, 8, 3) == (192, 256)
    assert [shard_streams(7, 3, r) for r in range(3)] == [(0, 3), (3, 5), (5, 7)]
    with pytest.raises(ValueError):
        shard_streams(2, 4, 0)


def test_two_rank_gradient_exchange_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict((r, (f, w)) for r, f, w in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_flats, ref_w = _reference_run(build_lstm(4, 5, 3))
    for r in (0, 1):
        flats, w = results[r]
        for a, b in zip(flats, ref_flats):
            assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max())
        assert np.abs(w - ref_w).max() <= 1e-12
    assert np.array_equal(results[0][1], results[1][1])  # replicas stay bit-identical


def test_bench_spawns_its_own_ranks_without_a_launcher():
    """`python bench.py --gpus 2` (no torchrun, no WORLD_SIZE) re-launches
    itself under torch.distributed.run; --dry-setup stops after the rank
    setup (gloo on CPU) so the launcher logic is tested without GPUs."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--dry-setup"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=repo)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(s) for s in out.stdout.splitlines() if s.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 for d in lines)
    assert sorted(tuple(d["streams"]) for d in lines) == [(0, 256), (256, 512)]
