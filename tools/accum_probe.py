"""Accuracy of the tensor-core GEMMs as a function of K (tools; GPU box).

    python tools/accum_probe.py

tcgen05 accumulates kind::tf32 products into fp32 TMEM with truncation
(round-toward-zero) when aligning the sum (as earlier tensor-core generations,
Fasi et al. 2021), so the relative error of one accumulator grows linearly in
the number of MMA accumulations -- visible at the dW depth of cfg4
(K = h * S = 16384).  Prints normwise error vs float64 for the dW form and the
NT form at several K, SIMT and tcgen05, coherent (all-positive) and random data.
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1503_02852_b200 import _lib  # noqa: E402


def main():
    L = _lib.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    rng = np.random.default_rng(0)
    m, n = 512, 512
    for kind in ("random", "coherent"):
        for k in (1024, 4096, 16384):
            if kind == "random":
                e = rng.uniform(-1, 1, size=(k, m)).astype(np.float32)
                y = rng.uniform(-1, 1, size=(k, n)).astype(np.float32)
            else:
                e = rng.uniform(0, 1, size=(k, m)).astype(np.float32)
                y = rng.uniform(0, 1, size=(k, n)).astype(np.float32)
            ref = e.astype(np.float64).T @ y.astype(np.float64)
            te, ty = torch.tensor(e, device="cuda"), torch.tensor(y, device="cuda")
            g = torch.empty((m, n), device="cuda")
            row = [f"{kind:8s} K={k:6d}"]
            for mode, name in ((1, "simt"), (3, "tc-dw")):
                _lib.check(L.rgb_gemm_dw(P(te), P(ty), P(g), m, n, k, ctypes.c_float(1.0), mode, st))
                torch.cuda.synchronize()
                err = np.abs(g.cpu().numpy() - ref).max() / np.abs(ref).max()
                row.append(f"{name} {err:.2e}")
            # NT form: C = A . B^T with A = e^T (m x k), B = y^T (n x k)
            a = torch.tensor(np.ascontiguousarray(e.T), device="cuda")
            b = torch.tensor(np.ascontiguousarray(y.T), device="cuda")
            c = torch.empty((m, n), device="cuda")
            _lib.check(L.rgb_gemm_nt_tma(P(a), P(b), P(b), P(c), m, n, k, st))
            torch.cuda.synchronize()
            err = np.abs(c.cpu().numpy() - ref).max() / np.abs(ref).max()
            row.append(f"tc-nt {err:.2e}")
            print("  ".join(row), flush=True)


if __name__ == "__main__":
    main()
