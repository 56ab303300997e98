"""Token-id input throughput (tuning aid): LSTM with a large input vocabulary
fed int64 ids -- no one-hot rows exist on the device.

    python tools/id_bench.py [vocab] [hidden] [streams]
"""
from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

import torch  # noqa: E402

import paper_1503_02852_b200 as P  # noqa: E402


def main():
    V = int(sys.argv[1]) if len(sys.argv) > 1 else 38000
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    S = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    net = P.build_lstm(V, H, 1000)
    w = P.Weights.init(net, 0)
    tr = P.Trainer(net, w, S, P.TrainConfig(h=32, h_prime=16, lr=1e-3, iterations=1))
    tr.enable_graphs(ids=True)
    gx, gt = tr.graph_inputs()
    for i in range(8):
        gx.copy_(torch.randint(0, V, (16 * S,), device="cuda"))
        gt.copy_(torch.randint(0, 1000, (16 * S,), device="cuda"))
        tr.step_graphed()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(10):
        tr.step_graphed()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"vocab {V} hidden {H} S {S}: {ms:.3f} ms/step, {16 * S / ms * 1e3:.0f} frames/s, loss {tr.loss():.3f}")


if __name__ == "__main__":
    main()
