"""Per-tensor parity diagnosis against the oracle (tools; runs on the GPU box).

    python tools/diag_parity.py --cfg cfg4 --streams 512 --iters 2 [--gemm-mode 0|1|2] [--eager]

Prints, per iteration, the normwise error of the output, every delta, every
eps and every dW by layer / connection name, worst first -- to find which
kernel of a configuration misses the 1e-4 bound.  Environment variables of the
library (RGB_PDL, RGB_TC_PAIR, RGB_TC_PERSIST, RGB_TC_CSPLIT, RGB_SCC_PDL,
RGB_WAVEFRONT) select kernel variants."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, os.path.join(REPO, "tests", "golden"))

import torch  # noqa: E402

import paper_1503_02852_b200 as P  # noqa: E402
from oracle import engine_np as O  # noqa: E402
from oracle_util import normwise  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg4")
    ap.add_argument("--streams", type=int, default=512)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--gemm-mode", type=int, default=0)
    ap.add_argument("--layers", type=int, default=3)
    ap.add_argument("--width", type=int, default=1024)
    ap.add_argument("--h", type=int, default=32)
    ap.add_argument("--hp", type=int, default=16)
    ap.add_argument("--eager", action="store_true")
    ap.add_argument("--top", type=int, default=12)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    from paper_1503_02852_b200 import _lib
    _lib.check(_lib.lib().rgb_set_gemm_mode(args.gemm_mode))
    W_ = args.width
    net = P.build_stacked_lstm(W_, [W_] * args.layers, W_)
    cg = P.condense(net)
    S, h, hp = args.streams, args.h, args.hp
    lin, lout = net.input_layers()[0], net.output_layers()[0]
    W = O.init_weights(net, 0)
    st_o = O.History(net, S, h)
    w = P.Weights(net, W)
    tr = P.Trainer(net, w, S, P.TrainConfig(h=h, h_prime=hp, lr=1e-3, iterations=1))
    if not args.eager:
        tr.enable_graphs()
        gx, gt = tr.graph_inputs()
    rng = np.random.default_rng(7)
    lname = {l.id: l.name for l in net.layers}
    cname = {c.id: f"{lname[c.src]}->{lname[c.dst]}(d{c.delay})" for c in net.connections}
    out_all = []
    for it in range(args.iters):
        x = rng.uniform(-1, 1, size=(hp * S, lin.size))
        t = rng.integers(0, lout.size, size=hp * S)
        if args.eager:
            tr.step(torch.tensor(x, dtype=torch.float32, device="cuda"), torch.tensor(t, device="cuda"))
        else:
            gx.copy_(torch.tensor(x, dtype=torch.float32))
            gt.copy_(torch.tensor(t))
            tr.step_graphed()
        torch.cuda.synchronize()
        out_o = O.forward_chunk(net, cg, W, st_o, x)
        cap = {}
        g_o = O.backward_window(net, cg, W, st_o, st_o.cursor, h, hp, O.inject_output_error(t, out_o), capture=cap)
        O.sgd_update(W, g_o, 1e-3)
        t1 = tr.state.cursor
        errs = {"out": normwise(tr.state.read_y(lout.id, t1 - hp + 1, t1).cpu().numpy(), out_o)}
        for lid in sorted(net.layer(l.id).id for l in net.layers):
            if lid in st_o.y and lid != lin.id:
                errs[f"y:{lname[lid]}"] = normwise(tr.state.read_y(lid, t1 - hp + 1, t1).cpu().numpy(),
                                                   st_o.y[lid][st_o.rows(t1 - hp + 1, t1)])
        delta, eps = P.window_errors(tr.state, t1, h)
        for k, v in cap["delta"].items():
            errs[f"delta:{lname[k]}"] = normwise(delta[k].cpu().numpy(), v)
        for k, v in cap["eps"].items():
            if net.layer(net.connection(k).dst).aggregation.value == "multiplicative":
                errs[f"eps:{cname[k]}"] = normwise(eps[k].cpu().numpy(), v)
        for cid, m in tr.grads.g.items():
            errs[f"dW:{cname[cid]}"] = normwise(m.cpu().numpy(), g_o[cid])
        worst = sorted(errs.items(), key=lambda kv: -kv[1])
        print(f"iter {it}: out {errs['out']:.2e}; worst:", flush=True)
        for k, v in worst[:args.top]:
            print(f"   {v:.3e}  {k}")
        out_all.append(errs)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out_all, f, indent=1)


if __name__ == "__main__":
    main()
