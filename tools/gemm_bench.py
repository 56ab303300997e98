"""Time the tcgen05 TMA GEMM on raw shapes (tuning aid).

    python tools/gemm_bench.py 512x2048x1024 512x1024x2048 8192x4096x1024
    python tools/gemm_bench.py --tf32 dw:4096x1024x16384   # plain-TF32 mode, dW form
"""
from __future__ import annotations

import ctypes
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

import torch  # noqa: E402

from paper_1503_02852_b200 import _lib  # noqa: E402


def lo(x):
    return x - (x.view(torch.int32) & ~0x1FFF).view(torch.float32)


def main():
    args = sys.argv[1:]
    if args and args[0].startswith("--lib="):
        # experiment variants built by tools/build_exp.sh, same ABI
        _lib._lib = None
        _lib.LIB_PATH = args.pop(0).split("=", 1)[1]
        print("library:", _lib.LIB_PATH)
    L = _lib.lib()
    if args and args[0] == "--tf32":
        args.pop(0)
        _lib.check(L.rgb_set_tc_precision(1))
        print("tensor-core precision: plain TF32")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    for shape in args:
        if shape.startswith("dw:"):  # G[m,n] = -E^T Y over k rows (the TMA-fed dW form)
            m, n, k = (int(v) for v in shape[3:].split("x"))
            e = torch.rand(k, m, device="cuda") * 2 - 1
            y = torch.rand(k, n, device="cuda") * 2 - 1
            g = torch.empty(m, n, device="cuda")
            run = lambda: L.rgb_gemm_dw(P(e), P(y), P(g), m, n, k, ctypes.c_float(-1.0), 3, st)  # noqa: E731
            for _ in range(3):
                _lib.check(run())
            torch.cuda.synchronize()
            ref = -(e.double().T @ y.double())
            err = ((g.double() - ref).abs().max() / ref.abs().max()).item()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                run()
            e1.record()
            torch.cuda.synchronize()
            us = 1000 * e0.elapsed_time(e1) / 20
            print(f"{shape}: {us:8.1f} us  {2 * m * n * k / us / 1e6:7.1f} TFLOP/s  err {err:.1e}")
            continue
        m, n, k = (int(v) for v in shape.split("x"))
        a = torch.rand(m, k, device="cuda") * 2 - 1
        b = torch.rand(n, k, device="cuda") * 2 - 1
        bl = lo(b)
        c = torch.empty(m, n, device="cuda")
        for _ in range(3):
            _lib.check(L.rgb_gemm_nt_tma(P(a), P(b), P(bl), P(c), m, n, k, st))
        torch.cuda.synchronize()
        ref = a.double() @ b.double().T
        err = ((c.double() - ref).abs().max() / ref.abs().max()).item()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        e0.record()
        for _ in range(reps):
            L.rgb_gemm_nt_tma(P(a), P(b), P(bl), P(c), m, n, k, st)
        e1.record()
        torch.cuda.synchronize()
        us = 1000 * e0.elapsed_time(e1) / reps
        print(f"{shape}: {us:8.1f} us  {2 * m * n * k / us / 1e6:7.1f} TFLOP/s  err {err:.1e}")
        if hasattr(L, "rgb_exp_trace"):  # per-stage clock64 trace of CTA 0 (RGB_EXP_TRACE build)
            import numpy as np
            buf = np.zeros((6, 1024), dtype=np.int64)
            L.rgb_exp_trace(buf.ctypes.data_as(ctypes.c_void_p))
            nst = int((buf[0] != 0).sum())
            t0 = buf[0, 0]
            rel = (buf[:, :nst] - t0)
            print("  stages", nst, "done at", buf[3, 0] - t0)
            for it in list(range(0, min(nst, 12))) + list(range(max(12, nst - 4), nst)):
                print(f"  it {it:4d} issue {rel[0, it]:8d} landed {rel[1, it]:8d} converted {rel[4, it]:8d} "
                      f"fenced {rel[5, it]:8d} mma {rel[2, it]:8d}")
            cta = np.zeros((1024, 4), dtype=np.int64)
            L.rgb_exp_cta(cta.ctypes.data_as(ctypes.c_void_p))
            nc = int((cta[:, 0] != 0).sum())
            c = cta[:nc, :3] - cta[:nc, 0].min()
            print(f"  ctas {nc}: start min/med/max {c[:,0].min()}/{int(np.median(c[:,0]))}/{c[:,0].max()} ns, "
                  f"mainloop {int(np.median(c[:,1]-c[:,0]))} (max {(c[:,1]-c[:,0]).max()}), "
                  f"epilogue {int(np.median(c[:,2]-c[:,1]))} (max {(c[:,2]-c[:,1]).max()}), last end {c[:,2].max()}")


if __name__ == "__main__":
    main()
