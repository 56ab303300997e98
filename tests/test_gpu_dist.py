"""The native multi-GPU exchange on one GPU: a world-size-1 NCCL communicator
created through the C ABI (rgb_comm_unique_id / rgb_comm_init), the flat
all-reduce, and the bucketed backward (rgb_backward_window_allreduce: per-
supernode dW buckets summed on a communication stream while the backward
continues) -- eagerly and inside captured CUDA graphs.  With one rank the sum
is the identity, so every result must equal the plain single-GPU step bit for
bit (dW tiles are computed in the same order in either schedule)."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1503_02852_b200 as P  # noqa: E402
from paper_1503_02852_b200 import _lib  # noqa: E402
from paper_1503_02852_b200.dist import NcclExchange  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def exchange():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    ex = NcclExchange(bucketed=True)
    yield ex
    torch.cuda.synchronize()
    ex.close()


def test_single_allreduce_exchange_equals_plain_step(exchange):
    """The default exchange: plain backward, then one NCCL all-reduce of the
    flat gradient through the C ABI (rgb_allreduce_grads)."""
    ex = NcclExchange.__new__(NcclExchange)
    ex.__dict__.update(exchange.__dict__)
    ex.bucketed = False
    net = P.build_lstm(64, 128, 64)
    cfg = P.TrainConfig(h=8, h_prime=4, lr=0.01, iterations=1)
    wa, wb = P.Weights.init(net, 1), P.Weights.init(net, 1)
    ta, tb = P.Trainer(net, wa, 16, cfg), P.Trainer(net, wb, 16, cfg)
    rng = np.random.default_rng(1)
    for _ in range(4):
        x = torch.tensor(rng.uniform(-1, 1, size=(64, 64)), dtype=torch.float32, device="cuda")
        t = torch.tensor(rng.integers(0, 64, size=64), device="cuda")
        ta.step(x, t)
        tb.step(x, t, ex)
        assert ta.loss() == tb.loss()
    assert torch.equal(wa.flat, wb.flat)
    ex.handle = None  # owned by the fixture


def test_comm_size_and_flat_allreduce(exchange):
    n, r = ctypes.c_int(), ctypes.c_int()
    _lib.check(_lib.lib().rgb_comm_size(exchange.handle, ctypes.byref(n), ctypes.byref(r)))
    assert (n.value, r.value) == (1, 0)
    x = torch.randn(1000003, device="cuda")
    y = x.clone()
    exchange.allreduce_(y)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    assert exchange.max_(3.5) == 3.5


@pytest.mark.parametrize("graphs", [False, True])
def test_bucketed_backward_equals_plain_step(exchange, graphs):
    net = P.build_stacked_lstm(256, [256, 256], 256)
    S = 64
    cfg = P.TrainConfig(h=16, h_prime=8, lr=0.01, iterations=1)
    wa, wb = P.Weights.init(net, 3), P.Weights.init(net, 3)
    ta, tb = P.Trainer(net, wa, S, cfg), P.Trainer(net, wb, S, cfg)
    if graphs:
        tb.enable_graphs(exchange)
        gx, gt = tb.graph_inputs()
    rng = np.random.default_rng(0)
    for _ in range(6):
        x = torch.tensor(rng.uniform(-1, 1, size=(8 * S, 256)), dtype=torch.float32, device="cuda")
        t = torch.tensor(rng.integers(0, 256, size=8 * S), device="cuda")
        ta.step(x, t)
        if graphs:
            gx.copy_(x)
            gt.copy_(t)
            tb.step_graphed()
        else:
            tb.step(x, t, exchange)
        assert ta.loss() == tb.loss()
        assert torch.equal(ta.grads.flat, tb.grads.flat)
    assert torch.equal(wa.flat, wb.flat)
