"""Per-frame phase timing of the persistent SCC kernel (trace build):

    tools/build_exp.sh trace -DRGB_EXP_TRACE
    python tools/trace_scc.py tools/_exp/trace.so cfg2
marks per step si: 1+5si before the CTA barrier, 2+5si after it and the
slot resolution starts, 3+5si A staged, 4+5si dots done, 5+5si step done.
"""
from __future__ import annotations

import ctypes
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_02852_b200 import _lib  # noqa: E402


def main():
    _lib.LIB_PATH = sys.argv[1]
    import bench
    import paper_1503_02852_b200 as P
    cfg = dict(bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "cfg2"], name="x")
    net = bench.build_net(cfg)
    w = P.Weights.init(net, 0)
    S = cfg["S"]
    tr = P.Trainer(net, w, S, P.TrainConfig(h=cfg["h"], h_prime=cfg["hp"], lr=cfg["lr"], iterations=1))
    x = torch.rand((cfg["hp"] * S, cfg["n_in"]), device="cuda") * 2 - 1
    t = torch.randint(0, cfg["n_out"], (cfg["hp"] * S,), device="cuda")
    for _ in range(3):
        tr.step(x, t)
    torch.cuda.synchronize()
    buf = np.zeros((64 * 16 + 8), dtype=np.int64)
    lib = ctypes.CDLL(sys.argv[1])
    lib.rgb_exp_scc_trace(buf.ctypes.data_as(ctypes.c_void_p))
    pro = buf[64 * 16:]
    print("prologue (cycles from entry): build", pro[1] - pro[0], "analysis", pro[2] - pro[0],
          "W cache", pro[3] - pro[0])
    buf = buf[:64 * 16].reshape(64, 16)
    for f in range(1, 6):
        row = buf[f]
        nz = np.nonzero(row)[0]
        base = row[0]
        print(f"frame {f}: " + " ".join(f"{k}:{row[k] - base}" for k in nz) + f"  next frame at {buf[f + 1][0] - base}")


if __name__ == "__main__":
    main()
