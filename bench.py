"""Benchmark: BPTT(h; h') training frames/s of the graph-RNN step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

A *step* is one training iteration: forward over h' new frames per stream,
fused softmax-xent error injection + loss, backward over the h-frame window,
weight gradients, (N > 1: NCCL all-reduce of the flat gradient), SGD and the
W^T refresh -- the reference's train_loop iteration (engine.py:732-758).
frames/s = h' * S_total / seconds per step (engine.py:751-757, cli.py:335-346).

``value`` is measured with inputs resident in HBM (a pool of device batches),
CUDA events on the launching stream, max over ranks.  ``e2e`` is the same
metric through the public API (Trainer.step = the C-ABI calls) with pinned
HOST inputs/targets copied in and the loss read back every step.  The CPU
baseline of record is the reference itself: rnngraph.train_loop (numba,
float64, every host thread) installed in oracle/_ref by oracle/build_ref.sh,
on a bounded stream sample of the same workload (oracle/ref_runner.py; the
float64 numpy oracle port stands in only when oracle/_ref is absent) -- the
only places bench.py executes oracle/.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

CONFIGS = {
    # BASELINE.json configs[0..4]
    "cfg1": dict(desc="1-layer LSTM 128 (peepholes, forget gate), 39 in/out, 1 stream, h=32, h'=16",
                 n_in=39, cells=[128], n_out=39, S=1, h=32, hp=16, lr=1e-3),
    "cfg2": dict(desc="2-layer LSTM 512, 512 in/out, 1 stream, h'=T=256, h=512",
                 n_in=512, cells=[512, 512], n_out=512, S=1, h=512, hp=256, lr=1e-3),
    "cfg3": dict(desc="2-layer LSTM 512, 512 in/out, 64 streams, h=32, h'=16",
                 n_in=512, cells=[512, 512], n_out=512, S=64, h=32, hp=16, lr=1e-3),
    "cfg4": dict(desc="3-layer LSTM 1024, 1024 in/out, 512 streams (sharded over the GPUs), h=32, h'=16",
                 n_in=1024, cells=[1024, 1024, 1024], n_out=1024, S=512, h=32, hp=16, lr=1e-3),
    "cfg5": dict(desc="custom graph RNN (mult. layers, d=1,2 edges), 39-128-39, 1 stream, h=32, h'=16",
                 custom=True, n_in=39, n_out=39, S=1, h=32, hp=16, lr=1e-3),
}
METRIC = "BPTT training frames/sec (LSTM, fwd+bwd+update) at 1/2/4/8 B200 vs CPU oracle"


def build_net(cfg):
    import paper_1503_02852_b200 as P
    if cfg.get("custom"):
        return P.build_custom_graph(cfg["n_in"], 128, cfg["n_out"])
    return P.build_stacked_lstm(cfg["n_in"], cfg["cells"], cfg["n_out"])


def algorithmic_flops(net, S, h, hp):
    """F_iter = S * sum_dense R*C*[2h' + 2(h-d)[src in Delta] + 2h[dst in Delta]]."""
    from paper_1503_02852_b200.netdef import Role
    delta = {l.id for l in net.layers if l.role is not Role.INPUT and net.anterior(l.id)}
    tot = 0
    for c in net.iter_dense():
        rc = net.layer(c.dst).size * net.layer(c.src).size
        tot += rc * (2 * hp + (2 * (h - c.delay) if c.src in delta else 0) + (2 * h if c.dst in delta else 0))
    return S * tot


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md)


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU arms (oracle)


def cpu_oracle_rate(cfg, n_streams, min_seconds=10.0, max_iters=12, warm=2, seed=0):
    """Oracle iterations/s on ``n_streams`` streams of the workload -> frames/s."""
    from oracle import engine_np as O
    import paper_1503_02852_b200 as P
    net = build_net(cfg)
    cg = P.condense(net)
    W = O.init_weights(net, seed)
    st = O.History(net, n_streams, cfg["h"])
    rng = np.random.default_rng(seed)
    hp = cfg["hp"]
    times = []
    for it in range(warm + max_iters):
        x = rng.uniform(-1, 1, size=(hp * n_streams, cfg["n_in"]))
        t = rng.integers(0, cfg["n_out"], size=hp * n_streams)
        t0 = time.perf_counter()
        O.train_step(net, cg, W, st, x, t, cfg["h"], cfg["lr"])
        dt = time.perf_counter() - t0
        if it >= warm:
            times.append(dt)
            if sum(times) >= min_seconds:
                break
    return hp * n_streams / (sum(times) / len(times)), len(times), sum(times)


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:  # noqa: BLE001
        pass
    return os.cpu_count() or 1


def cpu_sample_streams(cfg) -> int:
    """Bounded sample: streams of the workload the CPU arms run.  Every stream
    is an independent context and the CPU kernels' cost is
    linear in S, so a stream subset measures the same per-frame rate."""
    return {"cfg4": 16, "cfg3": 64, "cfg2": 1}.get(cfg["name"], cfg["S"])


def reference_rate(cfg, n_streams, warm, iters):
    """The reference's own train_loop (numba, float64, all host threads) from
    oracle/_ref on ``n_streams`` streams of the workload: (frames/s, cpu_baseline
    dict) or None when the reference is not installed on this box."""
    from oracle import ref_runner as RR
    if RR.load_reference() is None:
        return None
    net = build_net(cfg)
    rate, n, secs, _ = RR.time_train_loop(net, n_streams, cfg["h"], cfg["hp"], cfg["lr"], warm, iters)
    nb = RR.numba_info()
    return rate, {"value": rate, "unit": "frames/s", "cores": nb["threads"], "kind": "reference",
                  "sample": f"reference rnngraph.train_loop (oracle/_ref, numba {nb['numba']}, float64, "
                            f"NUMBA_NUM_THREADS={nb['threads']}, {RR.cpu_model()}) on {n_streams} of {cfg['S']} "
                            f"streams of {cfg['name']}, h={cfg['h']}, h'={cfg['hp']}: {n} iterations after {warm} "
                            f"warm-up, {secs:.1f} s"}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = cpu_sample_streams(cfg)
    if cfg["name"] == "cfg2":
        cfg = dict(cfg, hp=32, h=64)  # bounded: a 1/8 slice of the T=256 window
    got = reference_rate(cfg, n, max(args.warmup, math.ceil(cfg["h"] / cfg["hp"]) + 1), args.steps)
    if got is not None:
        value, cpu = got
    else:  # the reference is not installed here: the oracle port (float64 numpy)
        from oracle import engine_np as O
        import paper_1503_02852_b200 as P
        net = build_net(cfg)
        cg = P.condense(net)
        W = O.init_weights(net, 0)
        st = O.History(net, n, cfg["h"])
        rng = np.random.default_rng(0)
        rates = []
        for it in range(args.warmup + args.steps):
            x = rng.uniform(-1, 1, size=(cfg["hp"] * n, cfg["n_in"]))
            t = rng.integers(0, cfg["n_out"], size=cfg["hp"] * n)
            t0 = time.perf_counter()
            O.train_step(net, cg, W, st, x, t, cfg["h"], cfg["lr"])
            if it >= args.warmup:
                rates.append(cfg["hp"] * n / (time.perf_counter() - t0))
        value = len(rates) / sum(1.0 / r for r in rates)
        cpu = {"value": value, "unit": "frames/s", "cores": blas_threads(), "kind": "port",
               "sample": f"{n} of {cfg['S']} streams of {cfg['name']}, h={cfg['h']}, h'={cfg['hp']}, float64 numpy"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * cfg["hp"] * n / value,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": cfg["name"] + ": " + cfg["desc"]},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def paper_flops_per_frame(net) -> int:
    """The paper's operation count (reference cli.py:49-55, count_flops): 6 *
    rows * cols per dense connection per frame; identity edges and
    elementwise work count zero."""
    return 6 * sum(net.layer(c.dst).size * net.layer(c.src).size for c in net.iter_dense())


# ---------------------------------------------------------------------------
# our arm


def prof_snapshot(L):
    import ctypes
    out = {}
    for i, name in enumerate(("ew", "gemm", "gemm_frame", "ew_frame", "dw", "softmax", "inject", "sgd", "transpose",
                              "scc")):
        ms, n, fl, by = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        L.rgb_profile_read(i, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(fl), ctypes.byref(by))
        if n.value:
            out[name] = {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value}
    return out


def launches(L):
    import ctypes
    v = ctypes.c_int64()
    L.rgb_launch_count(ctypes.byref(v))
    return v.value


def measure_intra_stream(P, steps=2):
    """cfg2 single stream: hoisted (paper) vs frame-sequential (baseline) schedule."""
    import torch
    cfg = CONFIGS["cfg2"]
    net = build_net(dict(cfg, name="cfg2"))
    res = {}
    for label, fp in (("hoisted", True), ("sequential", False)):
        w = P.Weights.init(net, 0)
        tr = P.Trainer(net, w, 1, P.TrainConfig(h=cfg["h"], h_prime=cfg["hp"], lr=cfg["lr"], iterations=1,
                                                 frame_parallel=fp))
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.rand((cfg["hp"], cfg["n_in"]), device="cuda", generator=g) * 2 - 1
        t = torch.randint(0, cfg["n_out"], (cfg["hp"],), device="cuda", generator=g)
        for _ in range(3):  # fill the 512-frame window
            tr.step(x, t)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            tr.step(x, t)
        e1.record()
        torch.cuda.synchronize()
        res[label] = cfg["hp"] / (e0.elapsed_time(e1) / steps / 1000.0)
    from paper_1503_02852_b200.condense import condense
    frame_steps = sum(1 for sn in condense(net).nodes if sn.recurrent) * (cfg["hp"] + cfg["h"])
    step_us = 1e6 * cfg["hp"] / res["hoisted"]
    return {"workload": "cfg2: " + cfg["desc"], "hoisted_frames_per_s": res["hoisted"],
            "sequential_frames_per_s": res["sequential"], "speedup": res["hoisted"] / res["sequential"],
            "schedule": "hoisted SCC loops on the persistent kernel, the two layers pipelined over "
                        "frame blocks (cross-layer wavefront, SURVEY 8(f2))",
            # whole iteration / recurrent frame steps: with the layers overlapped
            # this is an effective figure, below the kernel's per-frame latency
            "us_per_recurrent_frame_step": step_us / frame_steps, "steps": steps}


def measure_tf32(P, L, cfg, S, value_fp32, steps=10):
    """The same cfg4 step with the tensor-core GEMMs in plain TF32
    (rgb_set_tc_precision(1): one kind::tf32 product per k-step instead of
    3xTF32).  A separately bounded precision mode (north_star; bound in
    tests/test_gpu_gemm.py), reported beside -- never as -- the fp32 headline."""
    import torch
    from paper_1503_02852_b200 import _lib
    h, hp = cfg["h"], cfg["hp"]
    net = build_net(cfg)
    _lib.check(L.rgb_set_tc_precision(1))
    try:
        tr = P.Trainer(net, P.Weights.init(net, 0), S, P.TrainConfig(h=h, h_prime=hp, lr=cfg["lr"], iterations=1))
        g = torch.Generator(device="cuda").manual_seed(4321)
        x = torch.rand((hp * S, cfg["n_in"]), device="cuda", generator=g) * 2 - 1
        t = torch.randint(0, cfg["n_out"], (hp * S,), device="cuda", generator=g)
        for _ in range(math.ceil(h / hp) + 1):
            tr.step(x, t)
        tr.enable_graphs(None)  # captured after the switch: the graphs hold the TF32 launches
        gx, gt = tr.graph_inputs()
        gx.copy_(x)
        gt.copy_(t)
        for _ in range(tr._cap // hp + 1):
            tr.step_graphed()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            tr.step_graphed()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
    finally:
        _lib.check(L.rgb_set_tc_precision(3))
    v = hp * S / (ms / 1000.0)
    return {"gemm_precision": "tf32 (1 tcgen05 product per k-step)", "frames_per_s": v, "ms_per_step": ms,
            "speedup_vs_3xtf32": v / value_fp32, "steps": steps,
            "bound": "normwise 2e-3 vs the float64 oracle per training step, operands rounded to nearest tf32 "
                     "(tests/test_gpu_gemm.py, BASELINE.md §5)"}


def measure_tf32_peak(seconds=2.0):
    """Dense TF32 tensor throughput of this GPU, measured like MEASURED_PEAKS.json's
    bf16 figure: cuBLAS fp32 matmul with TF32 allowed, 8192^3 (2*N^3 FLOP),
    best of 10 (burst) and back to back for ~`seconds` (sustained).  The fp32
    (3xTF32) ceiling of the tensor-core GEMMs is a third of it."""
    import torch
    n = 8192
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        c = torch.empty(n, n, device="cuda")
        for _ in range(3):
            torch.matmul(a, b, out=c)
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        reps = max(1, int(seconds * 1000.0 / best))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        sus = e0.elapsed_time(e1) / reps
        del a, b, c
        torch.cuda.empty_cache()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    flop = 2.0 * n ** 3
    return {"burst_tflops": flop / best / 1e9, "sustained_tflops": flop / sus / 1e9,
            "how": "cuBLAS fp32 matmul, TF32 allowed, 8192^3: best of 10 / back to back ~2 s (CUDA events)"}


def recurrent_summary(prof, steps, net, hp, h):
    from paper_1503_02852_b200.condense import condense
    n_scc = sum(1 for sn in condense(net).nodes if getattr(sn, "recurrent", False))
    frame_steps = n_scc * (hp + h)
    ms = sum(prof.get(k, {}).get("ms", 0.0) for k in ("gemm_frame", "ew_frame", "scc")) / steps
    return {"frame_steps_per_iter": frame_steps, "ms_per_iter": ms,
            "us_per_frame_step": 1000.0 * ms / frame_steps if frame_steps else None,
            "share_of_step": ms / max(1e-9, sum(v["ms"] for v in prof.values()) / steps)}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1503_02852_b200 as P
    from paper_1503_02852_b200 import _lib
    from paper_1503_02852_b200.dist import GradientExchange, NcclExchange, init_from_env, shard_streams

    rank, world, local = init_from_env("nccl")
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L = _lib.lib()
    _lib.check(L.rgb_set_tc_precision(1 if args.tc_precision == "tf32" else 3))
    ex = GradientExchange()  # timing max over ranks (torch.distributed plumbing)
    # the gradient exchange itself: NCCL through the C ABI, bucketed and
    # overlapped with the backward (rgb_backward_window_allreduce)
    nex = NcclExchange(bucketed=args.bucketed) if world > 1 else None
    S_total = cfg["S"] * (world if args.scaling == "weak" else 1)
    lo, hi = shard_streams(S_total, world, rank)
    S = hi - lo
    h, hp = cfg["h"], cfg["hp"]
    net = build_net(cfg)
    w = P.Weights.init(net, 0)  # identical on every rank (same seed)
    tr = P.Trainer(net, w, S, P.TrainConfig(h=h, h_prime=hp, lr=cfg["lr"], iterations=1))
    pool = 4
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    xs = [torch.rand((hp * S, cfg["n_in"]), device=dev, generator=g) * 2 - 1 for _ in range(pool)]
    ts = [torch.randint(0, cfg["n_out"], (hp * S,), device=dev, generator=g) for _ in range(pool)]
    exch = nex

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (also fills the h-frame window: ceil(h/h') iterations)
    nwarm = max(args.warmup, math.ceil(h / hp) + 1)
    for i in range(nwarm):
        n_before = launches(L)
        tr.step(xs[i % pool], ts[i % pool], exch)
        launches_per_step = launches(L) - n_before
    torch.cuda.synchronize()
    graphs = not args.no_graphs
    if graphs:
        # one captured graph per ring phase; warm them all up
        tr.enable_graphs(exch)
        gx, gt = tr.graph_inputs()
        for i in range(tr._cap // hp + 1):
            gx.copy_(xs[i % pool])
            gt.copy_(ts[i % pool])
            tr.step_graphed()
        torch.cuda.synchronize()

    def run_step(i, host=False):
        if graphs:
            src_x, src_t = (hx, ht) if host else (xs, ts)
            gx.copy_(src_x[i % pool], non_blocking=True)
            gt.copy_(src_t[i % pool], non_blocking=True)
            tr.step_graphed()
        else:
            tr.step((hx if host else xs)[i % pool], (ht if host else ts)[i % pool], exch)

    # (A) headline: device-resident inputs, CUDA events, max over ranks
    clocks = ClockSampler(local)
    with clocks:
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.steps):
            run_step(i)
        e1.record()
        torch.cuda.synchronize()
        barrier()
    # graph replays launch exactly the kernels an eager step launches
    n_launch = launches_per_step * args.steps
    ms = ex.max_(e0.elapsed_time(e1) / args.steps, dev)
    value = hp * S_total / (ms / 1000.0)

    # (B) profiled pass: per-launch CUDA events -> per-kernel device time
    L.rgb_profile_reset()
    L.rgb_profile_enable(1)
    for i in range(args.steps):
        tr.step(xs[i % pool], ts[i % pool], exch)
    L.rgb_profile_collect()
    L.rgb_profile_enable(0)
    prof = prof_snapshot(L)

    # (C) e2e through the public API with pinned HOST buffers + loss read-back.
    # Graph path: the next iteration's inputs are staged host->device on a
    # copy stream while the current one runs (Trainer.stage_inputs), and
    # every iteration's loss is read back to the host one iteration later
    # (Trainer.loss_async) -- all copies inside the timed region.
    hx = [x.cpu().pin_memory() for x in xs]
    ht = [t.cpu().pin_memory() for t in ts]
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if graphs:
        tr.stage_inputs(hx[0], ht[0])
        pending = None
        for i in range(args.steps):
            tr.step_graphed()
            fut = tr.loss_async()
            if i + 1 < args.steps:
                tr.stage_inputs(hx[(i + 1) % pool], ht[(i + 1) % pool])
            if pending is not None:
                pending()
            pending = fut
        pending()
    else:
        for i in range(args.steps):
            run_step(i, host=True)
            tr.loss()
    e2e_s = ex.max_((time.perf_counter() - t0) / args.steps, dev)
    e2e = {"value": hp * S_total / e2e_s, "unit": "frames/s",
           "h2d_bytes_per_step": int(hx[0].numel() * 4 + ht[0].numel() * 8), "d2h_bytes_per_step": 8}

    if rank != 0:
        return 0
    peaks = {}
    pk = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    tflops = float(peaks.get("bf16_tflops_sustained", 1400.0))
    peak_src = "measured" if peaks else "fallback"
    top = max(prof, key=lambda k: prof[k]["ms"])
    p = prof[top]
    per_launch_s = p["ms"] / 1000.0 / p["launches"]
    if p["flops"] > 0:
        achieved = p["flops"] / p["launches"] / per_launch_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tflops, "unit": "TFLOP/s", "frac": achieved / tflops}
    else:
        achieved = p["bytes"] / p["launches"] / per_launch_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm}
    traffic = None
    tpath = os.path.join(HERE, "profiles", "r02_traffic.json")
    if os.path.exists(tpath):  # committed ncu --set full capture (dram read + write per launch)
        with open(tpath) as f:
            traffic = json.load(f).get(top, {}).get("dram_bytes_per_launch")
    roof.update({"traffic": traffic, "kernel": top, "peak_source": peak_src + " (MEASURED_PEAKS.json)",
                 "share_of_step": p["ms"] / sum(v["ms"] for v in prof.values())})
    if roof["bound"] == "tensor":
        # fp32 work on tensor cores is 3xTF32: three kind::tf32 MMAs per fp32
        # product, so this dtype's ceiling is the MEASURED dense TF32 rate / 3
        terms = 1 if args.tc_precision == "tf32" else 3
        tf32 = measure_tf32_peak()
        roof["fp32_emulation"] = "3xTF32" if terms == 3 else "TF32"
        roof["tf32_peak_measured"] = tf32
        roof["fp32_ceiling"] = tf32["sustained_tflops"] / terms
        roof["frac_of_fp32_ceiling"] = achieved / roof["fp32_ceiling"]
    F_iter = algorithmic_flops(net, S_total, h, hp)
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic (U(-1,1) inputs, uniform class targets, "
                                                     "Weights.init seed 0)",
        "config": {"workload": cfg["name"] + ": " + cfg["desc"], "streams_total": S_total, "streams_per_gpu": S,
                   "h": h, "h_prime": hp, "global_batch_frames": hp * S_total,
                   "parallelism": (f"dp{world} (streams sharded; dW summed by NCCL through the C ABI, "
                                   + ("per-SCC buckets overlapped with the backward)" if args.bucketed
                                      else "one all-reduce after the backward)")) if world > 1 else "dp1",
                   "l2": "no flush: per-step working set (history + W + W^T + dW) exceeds the 126 MB L2",
                   "schedule": "hoisted (paper §3.1)",
                   "launch": "CUDA-graph replay per ring phase" if graphs else "eager",
                   "gemm_precision": args.tc_precision},
        "algorithmic_tflops": F_iter / (ms / 1000.0) / 1e12,
        # the two FLOP conventions: SURVEY §8(d)'s algorithmic unit (above) and
        # the paper's 6*R*C per dense edge per frame (reference cli.py:49-55)
        "paper_6rc": {"mflop_per_frame": paper_flops_per_frame(net) / 1e6,
                      "gflops": paper_flops_per_frame(net) * value / 1e9,
                      "e2e_gflops": paper_flops_per_frame(net) * e2e["value"] / 1e9},
        # the frame-sequential (recurrent) part of an iteration: device time of
        # the per-frame launches (or persistent SCC kernels) per frame step
        # (layers x frames of the forward chunk and the backward window)
        "recurrent": recurrent_summary(prof, args.steps, net, hp, h),
        "roofline": roof,
        "kernels": {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                        "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["flops"] else None,
                        "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["bytes"] else None}
                    for k, v in prof.items()},
        "e2e": e2e,
        "clocks": clocks.summary(),
        "gpu_launches": n_launch,
    }
    if world == 1 and not args.no_cpu:
        n = cpu_sample_streams(cfg)
        got = reference_rate(cfg, n, math.ceil(h / hp) + 1, 3)
        if got is not None:
            line["cpu_baseline"] = got[1]
        else:
            rate, iters, secs = cpu_oracle_rate(cfg, n, min_seconds=args.cpu_seconds)
            line["cpu_baseline"] = {"value": rate, "unit": "frames/s", "cores": blas_threads(), "kind": "port",
                                    "sample": f"oracle (float64 numpy) on {n} of {cfg['S']} streams of "
                                              f"{cfg['name']}, {iters} iterations after 2 warm-up, {secs:.1f} s"}
    if world == 1 and not args.no_intra:
        line["intra_stream"] = measure_intra_stream(P)
    if world == 1 and not args.no_tf32 and args.tc_precision != "tf32":
        line["tf32_mode"] = measure_tf32(P, L, cfg, S, value)
    print(json.dumps(line))
    if nex is not None:
        torch.cuda.synchronize()
        nex.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def dry_setup(args):
    """Rank setup only (CPU tests of the launcher): join the process group with
    gloo, shard the streams, print one JSON line per rank."""
    import torch.distributed as dist

    from paper_1503_02852_b200.dist import init_from_env, shard_streams
    cfg = dict(CONFIGS[args.config], name=args.config)
    rank, world, local = init_from_env("gloo")
    lo, hi = shard_streams(cfg["S"], world, rank)
    print(json.dumps({"dry_setup": True, "rank": rank, "world": world, "local_rank": local, "streams": [lo, hi]}),
          flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def relaunch(args, argv) -> int:
    """--gpus N > 1 without a launcher: re-run this script under
    torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1."""
    import socket
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-intra", action="store_true")
    ap.add_argument("--no-tf32", action="store_true", help="skip the plain-TF32 side measurement")
    ap.add_argument("--tc-precision", default="3xtf32", choices=["3xtf32", "tf32"],
                    help="tensor-core GEMM precision for the whole run (tf32: the separately bounded mode)")
    ap.add_argument("--no-graphs", action="store_true", help="eager launches instead of CUDA-graph replay")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--dry-setup", action="store_true", help="rank setup only (launcher test, CPU)")
    ap.add_argument("--bucketed", action="store_true",
                    help="N>1: bucketed backward with the all-reduce overlapped (DESIGN.md §8; off: one all-reduce)")
    raw = sys.argv[1:] if argv is None else list(argv)
    args = ap.parse_args(raw)
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args, raw)
    if args.dry_setup:
        return dry_setup(args)
    cfg = dict(CONFIGS[args.config], name=args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
