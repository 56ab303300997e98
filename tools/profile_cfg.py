"""Per-kernel-category device time of one training step of a bench config
(live CUDA events around every launch, the same profiler bench.py uses).

    python tools/profile_cfg.py --config cfg2 [--steps 2] [--seq] [--no-scc]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1503_02852_b200 as P  # noqa: E402
from paper_1503_02852_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--seq", action="store_true")
    ap.add_argument("--no-scc", action="store_true")
    ap.add_argument("--streams", type=int, default=None)
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config], name=args.config)
    S = args.streams or cfg["S"]
    L = _lib.lib()
    if args.no_scc:
        L.rgb_set_scc_mode(0)
    net = bench.build_net(cfg)
    w = P.Weights.init(net, 0)
    tr = P.Trainer(net, w, S, P.TrainConfig(h=cfg["h"], h_prime=cfg["hp"], lr=cfg["lr"], iterations=1,
                                             frame_parallel=not args.seq))
    x = torch.rand((cfg["hp"] * S, cfg["n_in"]), device="cuda") * 2 - 1
    t = torch.randint(0, cfg["n_out"], (cfg["hp"] * S,), device="cuda")
    for _ in range(-(-cfg["h"] // cfg["hp"]) + 1):
        tr.step(x, t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        tr.step(x, t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    L.rgb_profile_reset()
    L.rgb_profile_enable(1)
    for _ in range(args.steps):
        tr.step(x, t)
    L.rgb_profile_collect()
    L.rgb_profile_enable(0)
    prof = bench.prof_snapshot(L)
    out = {"config": args.config, "S": S, "ms_per_step": ms, "frames_per_s": cfg["hp"] * S / (ms / 1e3),
           "kernels": {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                           "us_per_launch": 1e3 * v["ms"] / v["launches"],
                           "tflops": v["flops"] / (v["ms"] / 1e3) / 1e12 if v["flops"] else None}
                       for k, v in prof.items()}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
