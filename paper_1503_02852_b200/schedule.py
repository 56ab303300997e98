"""Dependency analyser, part 2: the paper's intra-stream schedule as a GPU program.

``condense`` (condense.py) finds the supernodes; this module decides what runs
where on the device and emits the int32 program that the C executor
(csrc/rgb_plan.cu) interprets:

* Every connection that does not sit on a recurrent loop is **hoisted** out of
  the time loop: simple supernodes are evaluated once per chunk over all
  h'*S rows (forward) or h*S rows (backward), and the contributions that
  enter (forward) or leave (backward) a recurrent SCC from outside are
  precomputed over the whole chunk/window as one GEMM into a partial buffer.
  The reference instead evaluates *all* anteriors of SCC members per frame
  (engine.py:407-410, 570-573); the hoisted form is the paper's intent
  (§3.1) and only changes floating-point summation order.
* Only the intra-SCC edges stay in the per-frame loop (forward ascending,
  backward descending), with the members in the analyser's internal order.
* Adjacent work is packed into as few launches as the data dependencies
  allow: independent GEMM jobs share one grouped launch, and elementwise layer
  ops that only read what the same thread just produced are fused into a GEMM
  epilogue or an elementwise chain.  For a peephole LSTM this gives one launch
  per backward frame and two per forward frame.
* Weight gradients of every dense edge are one grouped dW launch over the
  whole window (Eq. 19, engine.py:578-599).
* ``sequential=True`` programs reproduce the reference's frame-by-frame mode
  (``frame_parallel=False``, engine.py:407/570) -- the paper's baseline for the
  intra-stream speed-up.

Device data layout (all fp32, row = frame * S + stream, leading dim = width):

* RING (per layer y, per dense edge into a multiplicative layer z): 2*cap
  frames, *mirrored* -- frame t lives at slots t mod cap and t mod cap + cap, so
  any run of <= cap consecutive frames is contiguous without a memmove
  (the reference shifts its history with a memmove, engine.py:251-265).
* WIN (per-layer delta, per-edge eps into multiplicative layers, backward
  partials): h + max_delay frames; frame t1 sits at index h-1 and the
  trailing max_delay frames stay zero, which realises eps(t + d) = 0 beyond t1
  (engine.py:527-529) without a branch.
* CHUNK (input staging, forward partials, injected output error): h frames.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .condense import CondensedGraph
from .netdef import Activation, Aggregation, NetworkDef, Role, WeightKind

__all__ = ["Program", "build_program", "EngineError"]

MAGIC = 0x52474231
HEADER = 32
RING, WIN, CHUNK = 0, 1, 2
STEP_EW, STEP_GEMM, STEP_SOFTMAX, STEP_LOOP, STEP_DW, STEP_AR = 1, 2, 3, 4, 5, 6
EW_FWD_ADD, EW_FWD_MUL, EW_CONST1, EW_BWD = 0, 1, 2, 3
ACT = {Activation.IDENTITY: 0, Activation.SIGMOID: 1, Activation.TANH: 2, Activation.SOFTMAX: 3}
MAX_TERMS, MAX_RANK1, MAX_FAC, MAX_CHAIN, MAX_SEGS, MAX_JOBS, MAX_CHAINS, MAX_DW = 4, 3, 4, 6, 4, 8, 8, 48
ACC = "acc"
ALIGN = 32  # floats (128 B) per buffer


class EngineError(RuntimeError):
    """Mirror of the reference ``EngineError`` (engine.py:86-87)."""


# ---------------------------------------------------------------------------
# workspace layout


@dataclass
class Layout:
    S: int
    h: int
    cap: int
    maxd: int
    bufs: list = field(default_factory=list)          # (kind, width, offset_floats, name)
    names: dict = field(default_factory=dict)
    w_off: dict = field(default_factory=dict)         # cid -> offset in flat W/WT/G
    n_params: int = 0
    ws_floats: int = 0
    scratch_off: int = 0

    def frames_of(self, kind: int) -> int:
        return 2 * self.cap if kind == RING else (self.h + self.maxd if kind == WIN else self.h)

    def add(self, name: str, kind: int, width: int) -> int:
        if name in self.names:
            return self.names[name]
        off = self.ws_floats
        self.bufs.append((kind, width, off, name))
        self.ws_floats = _align(off + self.frames_of(kind) * self.S * width)
        self.names[name] = len(self.bufs) - 1
        return self.names[name]


def _align(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


# ---------------------------------------------------------------------------
# items: one GEMM job or one elementwise op, with the buffers it reads/writes


@dataclass
class Op:
    kind: int
    act: int
    out: int
    width: int
    terms: list = field(default_factory=list)   # (buf, shift)
    rank1: list = field(default_factory=list)   # (buf, shift, cid)
    fac: list = field(default_factory=list)     # (buf, shift)
    y: tuple | None = None
    base: object = None                          # None | ACC | (buf, shift)
    inj: bool = False
    eps: list = field(default_factory=list)     # buf or -1 per factor

    def reads(self):
        r = [(b, s, False) for b, s in self.terms] + [(b, s, True) for b, s, _ in self.rank1]
        r += [(b, s, False) for b, s in self.fac]
        if self.y is not None:
            r.append((self.y[0], self.y[1], False))
        if isinstance(self.base, tuple):
            r.append((self.base[0], self.base[1], False))
        return r

    def writes(self):
        return [self.out] + [e for e in self.eps if e >= 0]


@dataclass
class Job:
    segs: list      # (buf, shift, cid, trans)
    ops: list       # epilogue chain; ops[0].base is ACC
    width: int

    def seg_reads(self):
        return [(b, s, False) for b, s, _, _ in self.segs]


@dataclass
class Softmax:
    buf: int


@dataclass
class Loop:
    reverse: bool
    body: list      # packed steps


@dataclass
class Dw:
    jobs: list      # (eps_buf, eps_shift, y_buf, y_shift, cid)


@dataclass
class AllReduce:
    ranges: list    # (first, last) float offsets into the flat gradient, [first, last)


# ---------------------------------------------------------------------------
# packing items into launches


class _Launch:
    def __init__(self, kind: str):
        self.kind = kind          # "G" or "E"
        self.units = []           # G: [Job]; E: [[Op, ...] chains]
        self.reads = []           # (buf, shift, rank1, owner)
        self.writes = {}          # buf -> owner


def _conflicts_new_unit(L: _Launch, reads, writes, single_frame: bool) -> bool:
    """A new job/chain (owner != any existing) must not read what the launch
    writes, nor write what the launch reads or writes."""
    for b, s, _ in reads:
        if b in L.writes:
            if not single_frame or s == 0:
                return True
    for b in writes:
        if b in L.writes:
            return True
        for rb, rs, _, _ in L.reads:
            if rb == b and (not single_frame or rs == 0):
                return True
    return False


def _can_join_chain(L: _Launch, owner: int, chain_width: int, op: Op, single_frame: bool) -> bool:
    if op.width != chain_width:
        return False
    for b, s, r1 in op.reads():
        if b in L.writes:
            if L.writes[b] == owner and s == 0 and not r1:
                continue  # element-local: produced by this thread earlier in the chain
            if single_frame and s != 0:
                continue  # a different frame's rows
            return False
    for b in op.writes():
        if b in L.writes:
            return False
        for rb, rs, _, ro in L.reads:
            if rb != b:
                continue
            if ro == owner and rs == 0:
                continue  # already consumed by this thread
            if single_frame and rs != 0:
                continue
            return False
    return True


def pack(items, single_frame: bool):
    """Greedy packing of items (in dependency order) into launches."""
    steps = []
    cur: _Launch | None = None

    def flush():
        nonlocal cur
        if cur is not None:
            steps.append(cur)
        cur = None

    for it in items:
        if isinstance(it, (Softmax, Loop, Dw, AllReduce)):
            flush()
            steps.append(it)
            continue
        if isinstance(it, Job):
            reads = it.seg_reads() + [r for op in it.ops for r in op.reads()]
            writes = [w for op in it.ops for w in op.writes()]
            if cur is not None and cur.kind == "G" and len(cur.units) < MAX_JOBS and not _conflicts_new_unit(
                    cur, reads, writes, single_frame):
                pass
            else:
                flush()
                cur = _Launch("G")
            owner = len(cur.units)
            cur.units.append(it)
            cur.reads += [(b, s, r1, owner) for b, s, r1 in reads]
            for w in writes:
                cur.writes[w] = owner
            continue
        op: Op = it
        placed = False
        if cur is not None:
            if cur.kind == "G":
                for owner, job in enumerate(cur.units):
                    if len(job.ops) < MAX_CHAIN and _can_join_chain(cur, owner, job.width, op, single_frame):
                        job.ops.append(op)
                        placed = True
                        break
            else:
                for owner, chain in enumerate(cur.units):
                    if len(chain) < MAX_CHAIN and _can_join_chain(cur, owner, chain[0].width, op, single_frame):
                        chain.append(op)
                        placed = True
                        break
                if not placed and len(cur.units) < MAX_CHAINS and not _conflicts_new_unit(
                        cur, op.reads(), op.writes(), single_frame):
                    cur.units.append([op])
                    owner = len(cur.units) - 1
                    placed = True
            if placed:
                cur.reads += [(b, s, r1, owner) for b, s, r1 in op.reads()]
                for w in op.writes():
                    cur.writes[w] = owner
        if not placed:
            flush()
            cur = _Launch("E")
            cur.units.append([op])
            cur.reads += [(b, s, r1, 0) for b, s, r1 in op.reads()]
            for w in op.writes():
                cur.writes[w] = 0
    flush()
    return steps


# ---------------------------------------------------------------------------
# encoding


def _enc_op(op: Op) -> list[int]:
    w = [op.kind, op.act, op.out, len(op.terms)]
    for b, s in op.terms:
        w += [b, s]
    w.append(len(op.rank1))
    for b, s, c in op.rank1:
        w += [b, s, c]
    w.append(len(op.fac))
    for b, s in op.fac:
        w += [b, s]
    w += list(op.y) if op.y is not None else [-1, 0]
    if op.base is None:
        w += [-1, 0]
    elif op.base == ACC:
        w += [-2, 0]
    else:
        w += list(op.base)
    w.append(1 if op.inj else 0)
    w.append(len(op.eps))
    w += list(op.eps)
    return w


def _enc_chain(ops) -> list[int]:
    w = [ops[0].width, len(ops)]
    for op in ops:
        w += _enc_op(op)
    return w


def encode(steps) -> list[int]:
    out: list[int] = []
    for st in steps:
        if isinstance(st, _Launch) and st.kind == "G":
            out += [STEP_GEMM, len(st.units)]
            for job in st.units:
                out.append(len(job.segs))
                for b, s, c, t in job.segs:
                    out += [b, s, c, t]
                out += _enc_chain(job.ops)
        elif isinstance(st, _Launch):
            out += [STEP_EW, len(st.units)]
            for chain in st.units:
                out += _enc_chain(chain)
        elif isinstance(st, Softmax):
            out += [STEP_SOFTMAX, st.buf]
        elif isinstance(st, Loop):
            body = encode(st.body)
            out += [STEP_LOOP, 1 if st.reverse else 0, len(body)] + body
        elif isinstance(st, Dw):
            for k in range(0, len(st.jobs), MAX_DW):
                part = st.jobs[k:k + MAX_DW]
                out += [STEP_DW, len(part)]
                for j in part:
                    out += list(j)
        elif isinstance(st, AllReduce):
            out += [STEP_AR, len(st.ranges)]
            for a, b in st.ranges:
                out += [*_split64(a), *_split64(b)]
        else:  # pragma: no cover
            raise TypeError(st)
    return out


# ---------------------------------------------------------------------------
# the analyser proper


@dataclass
class Program:
    words: np.ndarray              # int32 program for rgb_plan_create
    layout: Layout
    y_buf: dict                    # layer id -> ring buffer id
    in_buf: int
    out_buf: int
    stage_buf: int
    inj_buf: int
    softmax_feeds: str | None      # name of a softmax layer with posteriors (backward is an error)
    stats: dict                    # launch counts per phase (for DESIGN/bench reporting)


class _Emitter:
    def __init__(self, net: NetworkDef, cg: CondensedGraph, S: int, h: int, cap: int):
        self.net, self.cg = net, cg
        self.L = Layout(S=S, h=h, cap=cap, maxd=net.max_delay)
        L = self.L
        ins, outs = net.input_layers(), net.output_layers()
        if len(ins) != 1 or len(outs) != 1:
            raise EngineError(
                f"engine supports exactly one input and one output layer, got {len(ins)} and {len(outs)}")
        self.lin, self.lout = ins[0], outs[0]
        self.y = {l.id: L.add(f"y{l.id}", RING, l.size) for l in net.layers}
        self.z = {c.id: L.add(f"z{c.id}", RING, net.layer(c.dst).size) for c in net.connections
                  if self._mul(c.dst) and c.weight_kind is WeightKind.DENSE}
        self.stage = L.add("stage", CHUNK, self.lin.size)
        self.inj = L.add("inj", CHUNK, self.lout.size)
        self.has_delta = {l.id for l in net.layers if l.role is not Role.INPUT and net.anterior(l.id)}
        self.d = {lid: L.add(f"d{lid}", WIN, net.layer(lid).size) for lid in sorted(self.has_delta)}
        self.e = {c.id: L.add(f"e{c.id}", WIN, net.layer(c.dst).size) for c in net.connections if self._mul(c.dst)}
        self.node_of = cg.node_of_layer

    # helpers -----------------------------------------------------------
    def _mul(self, lid: int) -> bool:
        return self.net.layer(lid).aggregation is Aggregation.MULTIPLICATIVE

    def _same_scc(self, c) -> bool:
        n = self.node_of[c.src]
        return n == self.node_of[c.dst] and self.cg.nodes[n].recurrent

    def eps_ref(self, cid: int, shift: int):
        c = self.net.connection(cid)
        return (self.e[cid], shift) if self._mul(c.dst) else (self.d[c.dst], shift)

    def fac_ref(self, cid: int):
        c = self.net.connection(cid)
        if c.weight_kind is WeightKind.DENSE:
            return (self.z[cid], 0)
        return (self.y[c.src], -c.delay)

    def _act(self, lid: int) -> int:
        return ACT[self.net.layer(lid).activation]

    # forward ---------------------------------------------------------------
    def _sum_items(self, out_buf: int, width: int, act: int, segs, terms, rank1, base, kind=EW_FWD_ADD, **bwd):
        """Items computing out = act(base + sum segs + sum terms + sum rank1),
        spilling into partial buffers when a launch descriptor would overflow."""
        items = []
        segs, terms, rank1 = list(segs), list(terms), list(rank1)
        spill_id = 0
        while len(segs) > MAX_SEGS or len(terms) > MAX_TERMS - 1 or len(rank1) > MAX_RANK1:
            pbuf = self.L.add(f"spill{out_buf}_{spill_id}_{self._phase}", WIN if self._phase == "b" else CHUNK, width)
            spill_id += 1
            head_s, segs = segs[:MAX_SEGS], segs[MAX_SEGS:]
            head_t, terms = terms[:MAX_TERMS - 1], terms[MAX_TERMS - 1:]
            head_r, rank1 = rank1[:MAX_RANK1], rank1[MAX_RANK1:]
            if head_s and isinstance(base, tuple):
                head_t.append(base)
            op = Op(EW_FWD_ADD, ACT[Activation.IDENTITY], pbuf, width, terms=head_t, rank1=head_r,
                    base=ACC if head_s else base)
            items.append(Job(head_s, [op], width) if head_s else op)
            base = (pbuf, 0)
        if segs:
            t = terms + ([base] if isinstance(base, tuple) else [])
            op = Op(kind, act, out_buf, width, terms=t, rank1=rank1, base=ACC, **bwd)
            items.append(Job(segs, [op], width))
        else:
            items.append(Op(kind, act, out_buf, width, terms=terms, rank1=rank1, base=base, **bwd))
        return items

    def _fwd_layer(self, lid: int, which: str):
        """Forward items for one layer.  which: 'all' (every anterior), 'ext'
        (hoisted contributions from outside its SCC), 'int' (per-frame part)."""
        net = self.net
        layer = net.layer(lid)
        if layer.role is Role.INPUT:
            if which == "int":
                return []
            return [Op(EW_FWD_ADD, 0, self.y[lid], layer.size, terms=[(self.stage, 0)])]
        ants = net.anterior(lid)
        if not ants:
            return [] if which == "ext" else [Op(EW_CONST1, 0, self.y[lid], layer.size)]
        pick = lambda c: which == "all" or (which == "int") == self._same_scc(c)  # noqa: E731
        items = []
        if layer.aggregation is Aggregation.ADDITIVE:
            segs, terms, rank1 = [], [], []
            for cid in ants:
                c = net.connection(cid)
                if not pick(c):
                    continue
                if c.weight_kind is WeightKind.IDENTITY:
                    terms.append((self.y[c.src], -c.delay))
                elif net.layer(c.src).size == 1:
                    rank1.append((self.y[c.src], -c.delay, cid))
                else:
                    segs.append((self.y[c.src], -c.delay, cid, 0))
            act = self._act(lid)
            if layer.activation is Activation.SOFTMAX:
                act = ACT[Activation.IDENTITY]
            if which == "ext":
                if not segs:
                    self._folded[lid] = (terms, rank1)
                    return []
                pbuf = self.L.add(f"pf{lid}", CHUNK, layer.size)
                self._partial[lid] = pbuf
                return self._sum_items(pbuf, layer.size, ACT[Activation.IDENTITY], segs, terms, rank1, None)
            base = None
            if which == "int":
                if lid in self._partial:
                    base = (self._partial[lid], 0)
                ft, fr = self._folded.pop(lid, ([], []))
                terms, rank1 = ft + terms, fr + rank1
            items += self._sum_items(self.y[lid], layer.size, act, segs, terms, rank1, base)
            if layer.activation is Activation.SOFTMAX:
                items.append(Softmax(self.y[lid]))
            return items
        # multiplicative: z per dense anterior, then the product of all z (ascending cid)
        for cid in ants:
            c = net.connection(cid)
            if not pick(c) or c.weight_kind is WeightKind.IDENTITY:
                continue
            if net.layer(c.src).size == 1:
                items.append(Op(EW_FWD_ADD, 0, self.z[cid], layer.size, rank1=[(self.y[c.src], -c.delay, cid)]))
            else:
                items += self._sum_items(self.z[cid], layer.size, 0, [(self.y[c.src], -c.delay, cid, 0)], [], [], None)
        if which != "ext":
            if len(ants) > MAX_FAC:
                raise EngineError(f"multiplicative layer {layer.name!r} has more than {MAX_FAC} inputs")
            items.append(Op(EW_FWD_MUL, 0, self.y[lid], layer.size, fac=[self.fac_ref(c) for c in ants]))
        return items

    # backward --------------------------------------------------------------
    def _bwd_layer(self, lid: int, which: str):
        net = self.net
        if lid not in self.has_delta:
            return []
        layer = net.layer(lid)
        post = net.posterior(lid)
        if layer.activation is Activation.SOFTMAX and post:
            self.softmax_feeds = layer.name
        pick = lambda c: which == "all" or (which == "int") == self._same_scc(c)  # noqa: E731
        segs, terms = [], []
        for cid in post:
            c = net.connection(cid)
            if not pick(c):
                continue
            ref = self.eps_ref(cid, c.delay)
            if c.weight_kind is WeightKind.IDENTITY:
                terms.append(ref)
            else:
                segs.append((ref[0], ref[1], cid, 1))
        if which == "ext":
            if not segs:
                self._folded[lid] = (terms, [])
                return []
            pbuf = self.L.add(f"pb{lid}", WIN, layer.size)
            self._partial[lid] = pbuf
            return self._sum_items(pbuf, layer.size, ACT[Activation.IDENTITY], segs, terms, [], None)
        base = None
        if which == "int":
            if lid in self._partial:
                base = (self._partial[lid], 0)
            terms = self._folded.pop(lid, ([], []))[0] + terms
        ants = net.anterior(lid)
        mul = layer.aggregation is Aggregation.MULTIPLICATIVE
        if mul and len(ants) > MAX_FAC:
            raise EngineError(f"multiplicative layer {layer.name!r} has more than {MAX_FAC} inputs")
        extra = dict(
            y=(self.y[lid], 0) if layer.activation not in (Activation.IDENTITY, Activation.SOFTMAX) else None,
            inj=lid == self.lout.id,
            fac=[self.fac_ref(c) for c in ants] if mul else [],
            eps=[self.e[c] for c in ants] if mul else [],
        )
        return self._sum_items(self.d[lid], layer.size, self._act(lid), segs, terms, [], base, kind=EW_BWD, **extra)

    # programs ----------------------------------------------------------------
    def forward(self, sequential: bool):
        self._phase, self._partial, self._folded = "f", {}, {}
        topo = [self.cg.nodes[i] for i in self.cg.topo_order]
        if sequential:
            head = self._fwd_layer(self.lin.id, "all")
            body = []
            for node in topo:
                for lid in node.internal_order:
                    if lid != self.lin.id:
                        body += self._fwd_layer(lid, "all")
            return pack(head, False) + [Loop(False, pack(body, True))]
        items = []
        for node in topo:
            if not node.recurrent:
                items += self._fwd_layer(node.internal_order[0], "all")
                continue
            for lid in node.internal_order:
                items += self._fwd_layer(lid, "ext")
            body = []
            for lid in node.internal_order:
                body += self._fwd_layer(lid, "int")
            items.append(Loop(False, pack(body, True)))
        return pack(items, False)

    def _dw_jobs(self, conns):
        jobs = []
        for c in conns:
            e, s = self.eps_ref(c.id, 0)
            jobs.append((e, s, self.y[c.src], -c.delay, c.id))
        return jobs

    def _ar_ranges(self, conns):
        """Flat-gradient ranges of ``conns``, adjacent ones merged."""
        w_off, _ = weight_offsets(self.net)
        spans = sorted((w_off[c.id], w_off[c.id] + self.net.layer(c.dst).size * self.net.layer(c.src).size)
                       for c in conns)
        out = []
        for a, b in spans:
            if out and a <= _align4(out[-1][1]):
                out[-1] = (out[-1][0], max(out[-1][1], b))
            else:
                out.append((a, b))
        return out

    def backward_bucketed(self):
        """The hoisted backward with the weight gradients in buckets for the
        multi-GPU exchange.  Supernodes are visited in reverse
        topological order as in backward(); the dW of an edge can run once the
        supernode holding its destination is done (its eps are final there,
        engine.py:519-566).  Finished edges collect into a bucket that is
        flushed -- one grouped dW step, then an all-reduce marker over those
        edges' gradient ranges -- right before the next recurrent SCC loop, so
        the executor sums the bucket over the GPUs while that latency-bound
        frame loop runs; the last bucket follows the last supernode.  Every
        dense edge lands in exactly one bucket (cfg4: 4 buckets, top layer
        first)."""
        self._phase, self._partial, self._folded = "b", {}, {}
        self.softmax_feeds = None
        topo = [self.cg.nodes[i] for i in reversed(self.cg.topo_order)]
        items, pending, done = [], [], set()

        def flush():
            nonlocal pending
            if pending:
                items.append(Dw(self._dw_jobs(pending)))
                items.append(AllReduce(self._ar_ranges(pending)))
            pending = []

        for node in topo:
            if not node.recurrent:
                items += self._bwd_layer(node.internal_order[0], "all")
            else:
                for lid in reversed(node.internal_order):
                    items += self._bwd_layer(lid, "ext")
                body = []
                for lid in reversed(node.internal_order):
                    body += self._bwd_layer(lid, "int")
                flush()
                items.append(Loop(True, pack(body, True)))
            members = set(node.internal_order)
            conns = [c for c in self.net.iter_dense() if c.dst in members and c.id not in done]
            done.update(c.id for c in conns)
            pending += conns
        pending += [c for c in self.net.iter_dense() if c.id not in done]
        flush()
        return pack(items, False)

    def backward(self, sequential: bool):
        self._phase, self._partial, self._folded = "b", {}, {}
        self.softmax_feeds = None
        topo = [self.cg.nodes[i] for i in reversed(self.cg.topo_order)]
        items = []
        if sequential:
            body = []
            for node in topo:
                for lid in reversed(node.internal_order):
                    body += self._bwd_layer(lid, "all")
            items.append(Loop(True, pack(body, True)))
        else:
            for node in topo:
                if not node.recurrent:
                    items += self._bwd_layer(node.internal_order[0], "all")
                    continue
                for lid in reversed(node.internal_order):
                    items += self._bwd_layer(lid, "ext")
                body = []
                for lid in reversed(node.internal_order):
                    body += self._bwd_layer(lid, "int")
                items.append(Loop(True, pack(body, True)))
        dw = []
        for c in self.net.iter_dense():
            e, s = self.eps_ref(c.id, 0)
            dw.append((e, s, self.y[c.src], -c.delay, c.id))
        if dw:
            items.append(Dw(dw))
        return pack(items, False)


def _count(steps) -> dict:
    n = {"launches": 0, "loop_launches_per_frame": 0}
    for st in steps:
        if isinstance(st, Loop):
            n["loop_launches_per_frame"] += _count(st.body)["launches"]
        else:
            n["launches"] += 1
    return n


def weight_offsets(net: NetworkDef) -> tuple[dict, int]:
    """Flat W / WT / G layout: dense connections in ascending id, each
    (dst, src) matrix starting on a 16-byte boundary."""
    off, table = 0, {}
    for c in net.iter_dense():
        table[c.id] = off
        off += (net.layer(c.dst).size * net.layer(c.src).size + 3) // 4 * 4
    return table, off


def weights_program(net: NetworkDef) -> np.ndarray:
    """A program with only the weight table (for sgd_update / refresh)."""
    w_off, n_params = weight_offsets(net)
    hdr = [0] * HEADER
    hdr[0:14] = [MAGIC, 1, 1, 1, 1 + net.max_delay, net.max_delay, 0, len(net.connections), -1, -1, -1, -1, 0, 0]
    hdr[18:20] = _split64(n_params)
    words = list(hdr)
    for c in net.connections:
        if c.weight_kind is WeightKind.DENSE:
            words += [net.layer(c.dst).size, net.layer(c.src).size, *_split64(w_off[c.id])]
        else:
            words += [0, 0, 0, 0]
    return np.asarray(words, dtype=np.int32)


def build_program(net: NetworkDef, cg: CondensedGraph, S: int, h: int, chunk: int | None = None) -> Program:
    """Emit the device program for ``S`` streams and horizon ``h``.  ``chunk``
    (the usual h') rounds the ring capacity up to a multiple of it."""
    cap = h + net.max_delay
    if chunk:
        cap = -(-cap // chunk) * chunk
    em = _Emitter(net, cg, S, h, cap)
    fwd = em.forward(False)
    fwd_seq = em.forward(True)
    bwd_bkt = em.backward_bucketed()
    bwd = em.backward(False)
    softmax_feeds = em.softmax_feeds
    bwd_seq = em.backward(True)
    L = em.L
    L.w_off, L.n_params = weight_offsets(net)
    L.scratch_off = L.ws_floats
    tgt = _align(h * S * max(net.layer(em.lout.id).size, 2))
    L.ws_floats = L.scratch_off + tgt + _align(2 * h * S) + ALIGN
    sections = [encode(fwd), encode(bwd), encode(fwd_seq), encode(bwd_seq), encode(bwd_bkt)]
    hdr = [0] * HEADER
    hdr[0:14] = [MAGIC, 1, S, h, cap, net.max_delay, len(L.bufs), len(net.connections), em.y[em.lin.id],
                 em.stage, em.y[em.lout.id], em.inj, em.lin.size, em.lout.size]
    hdr[14:20] = [*_split64(L.scratch_off), *_split64(L.ws_floats), *_split64(L.n_params)]
    hdr[20:25] = [len(s) for s in sections]
    words = list(hdr)
    for kind, width, o, _ in L.bufs:
        words += [kind, width, *_split64(o)]
    for c in net.connections:
        if c.weight_kind is WeightKind.DENSE:
            words += [net.layer(c.dst).size, net.layer(c.src).size, *_split64(L.w_off[c.id])]
        else:
            words += [0, 0, 0, 0]
    for s in sections:
        words += s
    stats = {"forward": _count(fwd), "backward": _count(bwd), "forward_seq": _count(fwd_seq),
             "backward_seq": _count(bwd_seq), "backward_bucketed": _count(bwd_bkt),
             "buckets": [st.ranges for st in bwd_bkt if isinstance(st, AllReduce)]}
    return Program(words=np.asarray(words, dtype=np.int32), layout=L, y_buf=dict(em.y), in_buf=em.y[em.lin.id],
                   out_buf=em.y[em.lout.id], stage_buf=em.stage, inj_buf=em.inj, softmax_feeds=softmax_feeds,
                   stats=stats)


def _align4(v: int) -> int:
    return (v + 3) // 4 * 4


def _split64(v: int):
    v = int(v)
    lo = v & 0xFFFFFFFF
    hi = v >> 32
    if lo >= 1 << 31:
        lo -= 1 << 32
    return [lo, hi]
