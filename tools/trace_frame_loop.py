"""Phase trace of the persistent frame-loop kernel (tuning aid; trace build):

    tools/build_exp.sh fltrace -DRGB_FL_TRACE
    python tools/trace_frame_loop.py tools/_exp/fltrace.so [S]

Runs cfg4 steps eagerly, then one forward chunk (last traced launch = the top
layer's forward loop) and one backward window (last = the bottom layer's
backward loop), printing per frame of CTA 0 the microseconds spent in: wait for
the frame barrier (A ready) -> MMA done -> accumulator staged -> split-K
reduced -> chain done -> [elementwise start -> done]."""
from __future__ import annotations

import ctypes
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_02852_b200 import _lib  # noqa: E402


def dump(L, label, nframes):
    buf = np.zeros((64, 16), dtype=np.int64)
    L.rgb_exp_fl_trace(buf.ctypes.data_as(ctypes.c_void_p))
    buf = (buf * (1000.0 / 1.9)).astype(np.int64)  # SM cycles -> ps-like units (1.9 GHz) so /1000 = us
    print(f"== {label}: per frame (us) a_ready->mma_done, ->staged, ->reduced, ->chain, ->ew_start, ->ew_done, "
          f"->next a_ready")
    for f in range(nframes):
        r = buf[f]
        nxt = buf[f + 1][0] if f + 1 < nframes else 0
        d = lambda a, b: (b - a) / 1000.0 if a and b else float("nan")  # noqa: E731
        end = r[6] if r[6] else r[4]
        ops = " ".join(f"{(r[8 + k] - r[3]) / 1000.0:5.2f}" for k in range(6) if r[8 + k])
        if r[14]:
            last = max(r[8 + k] for k in range(6) if r[8 + k])
            ops += f" | again: {(r[14] - last) / 1000.0:5.2f} {(r[15] - r[14]) / 1000.0:5.2f}"
        print(f"  f{f:2d}  {d(r[0], r[1]):6.2f} {d(r[1], r[2]):6.2f} {d(r[2], r[3]):6.2f} {d(r[3], r[4]):6.2f} "
              f"{d(r[4], r[5]):6.2f} {d(r[5], r[6]):6.2f}   {d(end, nxt):6.2f}   total {d(r[0], nxt):6.2f}"
              f"   ops(us after reduce, last pass) {ops}"
              + (f"   preload wait {d(r[3], r[7]):6.2f}" if r[7] else ""))


def main():
    _lib.LIB_PATH = sys.argv[1]
    import bench
    import paper_1503_02852_b200 as P
    cfg = dict(bench.CONFIGS["cfg4"], name="cfg4")
    S = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["S"]
    net = bench.build_net(cfg)
    w = P.Weights.init(net, 0)
    tr = P.Trainer(net, w, S, P.TrainConfig(h=cfg["h"], h_prime=cfg["hp"], lr=cfg["lr"], iterations=1))
    x = torch.rand((cfg["hp"] * S, cfg["n_in"]), device="cuda") * 2 - 1
    t = torch.randint(0, cfg["n_out"], (cfg["hp"] * S,), device="cuda")
    for _ in range(4):
        tr.step(x, t)
    torch.cuda.synchronize()
    L = _lib.lib()
    cg = P.condense(net)
    out = P.forward_chunk(net, cg, w, tr.state, P.Batch(x, cfg["hp"], S))
    torch.cuda.synchronize()
    dump(L, "forward, top layer", cfg["hp"])
    d = P.inject_output_error(t, out, P.Criterion.CROSS_ENTROPY_SOFTMAX, P.Activation.SOFTMAX)
    P.backward_window(net, cg, w, tr.state, P.BpttWindow(tr.state.cursor, cfg["h"], cfg["hp"]), d)
    torch.cuda.synchronize()
    dump(L, "backward, bottom layer", cfg["h"])


if __name__ == "__main__":
    main()
