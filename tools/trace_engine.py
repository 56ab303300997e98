"""Stage trace of the last traced tensor-core GEMM launch inside a real
training step (tuning aid; needs a trace build of the library):

    tools/build_exp.sh trace128 -DRGB_EXP_TRACE -DRGB_EXP_TRACE_GRID=128
    python tools/trace_engine.py tools/_exp/trace128.so cfg4
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
    cfg = dict(bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "cfg4"], name="x")
    net = bench.build_net(cfg)
    w = P.Weights.init(net, 0)
    S = int(sys.argv[3]) if len(sys.argv) > 3 else cfg["S"]
    tr = P.Trainer(net, w, S, P.TrainConfig(h=cfg["h"], h_prime=cfg["hp"], lr=cfg["lr"], iterations=1))
    x = torch.rand((cfg["hp"] * S, cfg["n_in"]), device="cuda") * 2 - 1
    t = torch.randint(0, cfg["n_out"], (cfg["hp"] * S,), device="cuda")
    for _ in range(4):
        tr.step(x, t)
    torch.cuda.synchronize()
    L = _lib.lib()
    buf = np.zeros((6, 1024), dtype=np.int64)
    L.rgb_exp_trace(buf.ctypes.data_as(ctypes.c_void_p))
    nst = int((buf[0] != 0).sum())
    rel = buf[:, :nst] - buf[0, 0]
    print("stages", nst)
    for it in range(nst):
        print(f"  it {it:4d} issue {rel[0, it]:8d} landed {rel[1, it]:8d} converted {rel[4, it]:8d} mma {rel[2, it]:8d}")
    print("scalar epilogue path taken" if buf[3, 15] else "vector epilogue path")
    ops = buf[3, 16:24]
    ops = ops[ops != 0]
    if len(ops) > 1:
        print("epilogue ops (cycles, CTA 0 thread 0):", np.diff(ops).tolist())
    cta = np.zeros((1024, 6), dtype=np.int64)
    L.rgb_exp_cta(cta.ctypes.data_as(ctypes.c_void_p))
    nc = int((cta[:, 0] != 0).sum())
    c = cta[:nc, :6] - cta[:nc, 0].min()
    print(f"ctas {nc}: start max {c[:, 0].max()} ns, mainloop med {int(np.median(c[:, 1] - c[:, 0]))} "
          f"max {(c[:, 1] - c[:, 0]).max()}, phase-1 epilogue med {int(np.median(c[:, 2] - c[:, 1]))}, "
          f"phase-1 end max {c[:, 2].max()}, cluster reduce done med {int(np.median(c[:, 3]))} max {c[:, 3].max()}")
    print(f"slice epilogue done med {int(np.median(c[:, 4]))} max {c[:, 4].max()}, "
          f"final cluster barrier med {int(np.median(c[:, 5]))} max {c[:, 5].max()}")


if __name__ == "__main__":
    main()
