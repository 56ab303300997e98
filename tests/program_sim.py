"""TEST INFRASTRUCTURE: a float64 numpy interpreter of the schedule program.

Mirrors csrc/rgb_plan.cu (operand resolution, mirrored rings, window buffers,
loops, dW) and the kernels' per-element semantics, so the analyser's emitted
program can be checked against the oracle on a CPU-only box.  It is not a
product path: the engine never calls it.
"""
from __future__ import annotations

import numpy as np

from paper_1503_02852_b200 import schedule as SC


def _j64(lo, hi):
    return (int(lo) & 0xFFFFFFFF) | (int(hi) << 32)


def _act(a, x):
    if a == 1:
        return 1.0 / (1.0 + np.exp(-x))
    if a == 2:
        return np.tanh(x)
    return x


def _dact(a, y):
    if a == 1:
        return y * (1.0 - y)
    if a == 2:
        return 1.0 - y * y
    return np.ones_like(y)


class Sim:
    def __init__(self, words):
        w = [int(v) for v in words]
        assert w[0] == SC.MAGIC
        self.S, self.h, self.cap, self.maxd = w[2:6]
        nb, nw = w[6], w[7]
        self.in_buf, self.stage_buf, self.out_buf, self.inj_buf, self.n_in, self.n_out = w[8:14]
        self.ws_floats = _j64(w[16], w[17])
        self.n_params = _j64(w[18], w[19])
        lens = w[20:25]
        pos = SC.HEADER
        self.bufs = []
        for _ in range(nb):
            self.bufs.append((w[pos], w[pos + 1], _j64(w[pos + 2], w[pos + 3])))
            pos += 4
        self.wts = []
        for _ in range(nw):
            self.wts.append((w[pos], w[pos + 1], _j64(w[pos + 2], w[pos + 3])))
            pos += 4
        self.prog = []
        for n in lens:
            self.prog.append(w[pos:pos + n])
            pos += n
        self.ws = np.zeros(self.ws_floats)
        self.cursor = 0

    # ------------------------------------------------------------------
    def _index(self, ctx, buf, shift, frames):
        kind, width, off = self.bufs[buf]
        t = ctx["t_a"] + shift
        if kind == SC.RING:
            assert t > self.cursor - self.cap and t + frames - 1 <= self.cursor, (buf, t, frames, self.cursor)
            idx = t % self.cap
        elif kind == SC.WIN:
            idx = t - ctx["t1"] + self.h - 1
            assert 0 <= idx and idx + frames <= self.h + self.maxd, (buf, idx)
        else:
            idx = t - ctx["chunk_base"]
            assert 0 <= idx and idx + frames <= self.h, (buf, idx)
        return off + idx * self.S * width, width

    def view(self, ctx, buf, shift, frames):
        o, width = self._index(ctx, buf, shift, frames)
        return self.ws[o:o + frames * self.S * width].reshape(frames * self.S, width)

    def write(self, ctx, buf, frames, val):
        kind, width, off = self.bufs[buf]
        o, _ = self._index(ctx, buf, 0, frames)
        self.ws[o:o + val.size] = val.ravel()
        if kind == SC.RING:
            S = self.S
            p0 = ctx["t_a"] % self.cap
            for f in range(frames):
                q = p0 + f  # physical slot of the primary copy, in [0, 2 cap)
                other = q + self.cap if q < self.cap else q - self.cap
                src = val[f * S:(f + 1) * S].ravel()
                mo = off + other * S * width
                self.ws[mo:mo + src.size] = src

    def wmat(self, ctx, cid, trans):
        rows, cols, off = self.wts[cid]
        if trans:
            return ctx["wt"][off:off + rows * cols].reshape(cols, rows)
        return ctx["w"][off:off + rows * cols].reshape(rows, cols)

    # ------------------------------------------------------------------
    def _op(self, rd, ctx):
        nxt = rd.__next__
        kind, act, out = nxt(), nxt(), nxt()
        terms = [(nxt(), nxt()) for _ in range(nxt())]
        rank1 = [(nxt(), nxt(), nxt()) for _ in range(nxt())]
        fac = [(nxt(), nxt()) for _ in range(nxt())]
        y = (nxt(), nxt())
        base = (nxt(), nxt())
        inj = nxt()
        eps = [nxt() for _ in range(nxt())]
        return dict(kind=kind, act=act, out=out, terms=terms, rank1=rank1, fac=fac, y=y, base=base, inj=inj, eps=eps)

    def _chain(self, rd, ctx):
        width, nops = next(rd), next(rd)
        return width, [self._op(rd, ctx) for _ in range(nops)]

    def _exec_op(self, op, ctx, acc):
        F = ctx["frames"]
        rows = F * self.S
        V = lambda b, s: self.view(ctx, b, s, F)  # noqa: E731
        k = op["kind"]
        if k == SC.EW_CONST1:
            width = self.bufs[op["out"]][1]
            self.write(ctx, op["out"], F, np.ones((rows, width)))
            return
        if k == SC.EW_FWD_MUL:
            v = V(*op["fac"][0]).copy()
            for b, s in op["fac"][1:]:
                v = v * V(b, s)
            self.write(ctx, op["out"], F, v)
            return
        width = self.bufs[op["out"]][1]
        if acc is not None:
            v = acc.copy()
        elif op["base"][0] >= 0:
            v = V(*op["base"]).copy()
        else:
            v = np.zeros((rows, width))
        for b, s in op["terms"]:
            v = v + V(b, s)
        if k == SC.EW_FWD_ADD:
            for b, s, cid in op["rank1"]:
                wcol = self.wmat(ctx, cid, 0)[:, 0]
                v = v + V(b, s)[:, 0:1] * wcol[None, :]
            self.write(ctx, op["out"], F, _act(op["act"], v))
            return
        assert k == SC.EW_BWD
        if op["act"] != 3:
            yv = V(*op["y"]) if op["y"][0] >= 0 else np.ones_like(v)
            v = v * (_dact(op["act"], yv) if op["y"][0] >= 0 else 1.0)
        if op["inj"]:
            lo = max(ctx["t_a"], ctx["t0"] + 1)
            hi = ctx["t_a"] + F - 1
            if lo <= hi:
                c2 = dict(ctx, t_a=lo)
                inj = self.view(c2, self.inj_buf, 0, hi - lo + 1)
                r0 = (lo - ctx["t_a"]) * self.S
                v[r0:] = v[r0:] + inj
        self.write(ctx, op["out"], F, v)
        facs = [V(b, s) for b, s in op["fac"]]
        for i, e in enumerate(op["eps"]):
            if e < 0:
                continue
            p = v.copy()
            for kk, f in enumerate(facs):
                if kk != i:
                    p = p * f
            self.write(ctx, e, F, p)

    def run(self, prog, ctx):
        rd = iter(prog)
        for kind in rd:
            F = ctx["frames"]
            if kind == SC.STEP_EW:
                chains = [self._chain(rd, ctx) for _ in range(next(rd))]
                for _, ops in chains:
                    for op in ops:
                        self._exec_op(op, ctx, None)
            elif kind == SC.STEP_GEMM:
                njobs = next(rd)
                jobs = []
                for _ in range(njobs):
                    segs = [(next(rd), next(rd), next(rd), next(rd)) for _ in range(next(rd))]
                    jobs.append((segs, self._chain(rd, ctx)))
                for segs, (width, ops) in jobs:
                    acc = np.zeros((F * self.S, width))
                    for b, s, cid, tr in segs:
                        acc += self.view(ctx, b, s, F) @ self.wmat(ctx, cid, tr).T
                    for i, op in enumerate(ops):
                        self._exec_op(op, ctx, acc if i == 0 else None)
            elif kind == SC.STEP_SOFTMAX:
                b = next(rd)
                x = self.view(ctx, b, 0, F)
                e = np.exp(x - x.max(axis=1, keepdims=True))
                self.write(ctx, b, F, e / e.sum(axis=1, keepdims=True))
            elif kind == SC.STEP_LOOP:
                rev, n = next(rd), next(rd)
                body = [next(rd) for _ in range(n)]
                order = range(F - 1, -1, -1) if rev else range(F)
                for f in order:
                    self.run(body, dict(ctx, t_a=ctx["t_a"] + f, frames=1))
            elif kind == SC.STEP_DW:
                for _ in range(next(rd)):
                    eb, es, yb, ys, cid = (next(rd) for _ in range(5))
                    E = self.view(ctx, eb, es, F)
                    Y = self.view(ctx, yb, ys, F)
                    rows, cols, off = self.wts[cid]
                    ctx["g"][off:off + rows * cols] = (-(E.T @ Y)).ravel()
                    ctx.setdefault("dw_written", []).append((off, off + rows * cols))
            elif kind == SC.STEP_AR:
                # the executor sums these ranges over the GPUs at this point:
                # record them with the dW ranges written so far
                ranges = [(_j64(next(rd), next(rd)), _j64(next(rd), next(rd))) for _ in range(next(rd))]
                ctx.setdefault("ar", []).append((ranges, list(ctx.get("dw_written", []))))
            else:
                raise AssertionError(kind)

    # ------------------------------------------------------------------ API
    def forward(self, w, x, sequential=False):
        F = x.shape[0] // self.S
        _, wd, off = self.bufs[self.stage_buf]
        self.ws[off:off + x.size] = x.ravel()
        self.cursor += F
        ctx = dict(t_a=self.cursor - F + 1, frames=F, chunk_base=self.cursor - F + 1, t1=self.cursor,
                   t0=self.cursor, w=w, wt=None, g=None)
        self.run(self.prog[2 if sequential else 0], ctx)
        return self.view(ctx, self.out_buf, 0, F).copy()

    def set_injection(self, d):
        _, _, off = self.bufs[self.inj_buf]
        self.ws[off:off + d.size] = d.ravel()

    def backward(self, wt, g, h, hp, sequential=False, bucketed=False):
        t1 = self.cursor
        ctx = dict(t_a=t1 - h + 1, frames=h, chunk_base=t1 - hp + 1, t1=t1, t0=t1 - hp, w=None, wt=wt, g=g)
        self.run(self.prog[4 if bucketed else (3 if sequential else 1)], ctx)
        return ctx


def flat_weights(prog, W: dict):
    """dict cid -> (rows, cols) matrix  ->  flat W and WT in the program layout."""
    L = prog.layout
    w = np.zeros(L.n_params)
    wt = np.zeros(L.n_params)
    for cid, m in W.items():
        o = L.w_off[cid]
        w[o:o + m.size] = m.ravel()
        wt[o:o + m.size] = m.T.ravel()
    return w, wt


def unflat(prog, net, flat):
    L = prog.layout
    out = {}
    for c in net.iter_dense():
        r, k = net.layer(c.dst).size, net.layer(c.src).size
        out[c.id] = flat[L.w_off[c.id]:L.w_off[c.id] + r * k].reshape(r, k)
    return out
