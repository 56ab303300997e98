"""One GPU's share of the strong-scaling run (tools; GPU box).

    python tools/share_probe.py [S ...]

cfg4 with S streams on this GPU: graph-replayed step time with no exchange,
with the default exchange (plain backward + one NCCL all-reduce) and with the
bucketed backward + NCCL exchange (world size 1: the schedule and stream
fork/join of the multi-GPU step, no peer traffic)."""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1503_02852_b200 as P  # noqa: E402
from paper_1503_02852_b200.dist import NcclExchange  # noqa: E402


def step_ms(S, exchange, steps=20):
    cfg = dict(bench.CONFIGS["cfg4"], name="cfg4")
    net = bench.build_net(cfg)
    tr = P.Trainer(net, P.Weights.init(net, 0), S, P.TrainConfig(h=32, h_prime=16, lr=1e-3, iterations=1))
    tr.enable_graphs(exchange)
    gx, gt = tr.graph_inputs()
    gx.copy_(torch.rand_like(gx) * 2 - 1)
    gt.copy_(torch.randint(0, 1024, gt.shape, device="cuda"))
    for _ in range(6):
        tr.step_graphed()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        tr.step_graphed()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [64, 128, 256, 512]
    ex = NcclExchange()
    exb = NcclExchange(bucketed=True)
    out = {}
    for S in sizes:
        out[S] = {"plain_ms": step_ms(S, None), "allreduce_nccl1_ms": step_ms(S, ex),
                  "bucketed_nccl1_ms": step_ms(S, exb)}
        print(S, out[S], flush=True)
    torch.cuda.synchronize()
    ex.close()
    exb.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
