"""Kernel-level parity of the two GEMM engines (SIMT fp32 and tcgen05 3xTF32)
against float64 numpy, through the C ABI's stand-alone GEMM entry points, and
full-engine parity with every GEMM forced onto the tensor cores."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle_util import normwise  # noqa: E402

import paper_1503_02852_b200 as P  # noqa: E402
from paper_1503_02852_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPES = [(128, 256, 32), (256, 512, 1024), (200, 300, 70), (1, 64, 512), (77, 39, 39), (1024, 2048, 1024),
          (513, 130, 257)]


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("m,n,k", SHAPES)
def test_gemm_nt(mode, m, n, k):
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    a = rng.uniform(-1, 1, size=(m, k))
    b = rng.uniform(-1, 1, size=(n, k))
    ta = torch.tensor(a, dtype=torch.float32, device="cuda")
    tb = torch.tensor(b, dtype=torch.float32, device="cuda")
    tc = torch.full((m, n), float("nan"), device="cuda")
    _lib.check(_lib.lib().rgb_gemm_nt(ctypes.c_void_p(ta.data_ptr()), ctypes.c_void_p(tb.data_ptr()),
                                      ctypes.c_void_p(tc.data_ptr()), m, n, k, mode, _stream()))
    ref = a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T
    err = normwise(tc.cpu().numpy(), ref)
    assert err < 1e-5, err


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("m,n,k", SHAPES)
def test_gemm_dw(mode, m, n, k):
    rng = np.random.default_rng(m + n + k)
    e = rng.uniform(-1, 1, size=(k, m))
    y = rng.uniform(-1, 1, size=(k, n))
    te = torch.tensor(e, dtype=torch.float32, device="cuda")
    ty = torch.tensor(y, dtype=torch.float32, device="cuda")
    tg = torch.full((m, n), float("nan"), device="cuda")
    _lib.check(_lib.lib().rgb_gemm_dw(ctypes.c_void_p(te.data_ptr()), ctypes.c_void_p(ty.data_ptr()),
                                      ctypes.c_void_p(tg.data_ptr()), m, n, k, ctypes.c_float(-1.0), mode,
                                      _stream()))
    ref = -(e.astype(np.float32).astype(np.float64).T @ y.astype(np.float32).astype(np.float64))
    err = normwise(tg.cpu().numpy(), ref)
    assert err < 1e-5, err


def test_engine_parity_with_tensor_cores_forced():
    """Every GEMM of the step (hoisted, per-frame, dW) on tcgen05."""
    from test_gpu_engine import run_pair
    L = _lib.lib()
    _lib.check(L.rgb_set_gemm_mode(2))
    try:
        assert run_pair(P.build_lstm(39, 128, 39), 2, 32, 16, 4, 1e-3, 0) < 1e-4
        assert run_pair(P.build_custom_graph(), 3, 16, 8, 4, 1e-3, 1) < 1e-4
        assert run_pair(P.build_stacked_lstm(64, [96, 64], 48), 5, 12, 4, 4, 1e-2, 2) < 1e-4
        assert run_pair(P.build_elman(5, 7, 6), 3, 6, 3, 4, 0.05, 3) < 1e-4
    finally:
        _lib.check(L.rgb_set_gemm_mode(0))


def test_engine_parity_simt_forced():
    from test_gpu_engine import run_pair
    L = _lib.lib()
    _lib.check(L.rgb_set_gemm_mode(1))
    try:
        assert run_pair(P.build_stacked_lstm(256, [256, 256], 256), 64, 8, 4, 3, 1e-3, 4) < 1e-4
    finally:
        _lib.check(L.rgb_set_gemm_mode(0))


def test_engine_parity_without_persistent_scc():
    """Per-frame launches instead of the persistent SCC kernel (the default)."""
    from test_gpu_engine import run_pair
    L = _lib.lib()
    _lib.check(L.rgb_set_scc_mode(0))
    try:
        assert run_pair(P.build_lstm(39, 128, 39), 1, 32, 16, 4, 1e-3, 0) < 1e-4
        assert run_pair(P.build_custom_graph(), 2, 16, 8, 4, 1e-3, 1) < 1e-4
    finally:
        _lib.check(L.rgb_set_scc_mode(1))


def test_persistent_scc_matches_per_frame_launches():
    """Same step with and without the persistent kernel (fp32 rounding only)."""
    from test_gpu_engine import run_pair
    net = P.build_stacked_lstm(48, [64, 64], 40)
    assert run_pair(net, 3, 24, 8, 5, 1e-2, 7) < 1e-4
    assert run_pair(P.build_custom_graph(16, 512, 16), 1, 32, 16, 3, 1e-3, 8) < 1e-4


@pytest.mark.parametrize("n_hidden,S", [(64, 24), (1024, 2), (42, 40)])
def test_persistent_scc_layouts(n_hidden, S):
    """Persistent SCC kernel layouts: several stream rows per CTA (register-
    blocked float4 dots), a W_rec too large for one cluster (grid-barrier
    fallback over many CTAs), an odd width (K not a multiple of 4, uneven
    column split).  The persistent kernel must actually run."""
    import ctypes
    from test_gpu_engine import run_pair
    L = _lib.lib()
    L.rgb_profile_reset()
    L.rgb_profile_enable(1)
    try:
        assert run_pair(P.build_lstm(8, n_hidden, 6), S, 8, 4, 2, 0.05, 31) < 1e-4
        L.rgb_profile_collect()
    finally:
        L.rgb_profile_enable(0)
    ms, n, fl, by = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    L.rgb_profile_read(9, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(fl), ctypes.byref(by))
    assert n.value > 0, "persistent SCC kernel did not run"


@pytest.mark.parametrize("wavefront", [1, 0])
def test_wavefront_matches_oracle(wavefront):
    """Cross-layer wavefront (default on): the stages between
    persistent SCC loops of the forward and backward sections run on their
    own streams over frame blocks; both schedules match the oracle."""
    from test_gpu_engine import run_pair
    L = _lib.lib()
    _lib.check(L.rgb_set_wavefront(wavefront))
    try:
        assert run_pair(P.build_stacked_lstm(24, [64, 64, 48], 20), 1, 96, 64, 3, 1e-2, 13) < 1e-4
        assert run_pair(P.build_stacked_lstm(16, [32, 32], 16), 3, 64, 48, 3, 1e-2, 14) < 1e-4
    finally:
        _lib.check(L.rgb_set_wavefront(1))


def test_wavefront_with_per_frame_tensor_core_loops():
    """The wavefront over loops of per-frame launches (no persistent kernel,
    S <= 128): tcgen05 per-frame GEMMs of two layers run on two streams."""
    from test_gpu_engine import run_pair
    L = _lib.lib()
    _lib.check(L.rgb_set_scc_mode(0))
    try:
        assert run_pair(P.build_stacked_lstm(64, [512, 512], 32), 64, 32, 16, 2, 1e-3, 21) < 1e-4
    finally:
        _lib.check(L.rgb_set_scc_mode(1))


@pytest.mark.parametrize("S,widths,h,hp", [(1, [40, 56, 24], 96, 64), (5, [64, 64], 80, 64), (40, [96, 96], 64, 32)])
def test_stacked_default_schedule_sweep(S, widths, h, hp):
    """Default engine (persistent SCC row blocks, forwarded chain values,
    template images, cross-layer wavefront) on stacked LSTMs of odd widths,
    several stream counts and window shapes, against the oracle."""
    from test_gpu_engine import run_pair
    # lr / S: gradients are raw sums over streams and frames (README.md:84-89),
    # a fixed lr diverges at 40 streams within three iterations
    assert run_pair(P.build_stacked_lstm(12, widths, 10), S, h, hp, 3, 1e-2 / S, 31 + S) < 1e-4


def test_engine_parity_large_auto():
    """cfg3-like shapes, where auto mode routes the big GEMMs to tcgen05."""
    from test_gpu_engine import run_pair
    assert run_pair(P.build_stacked_lstm(512, [512, 512], 512), 64, 32, 16, 3, 1e-3, 5) < 1e-4


TMA_SHAPES = [(512, 4096, 1024),   # 128 tiles of 128, no split
              (512, 1024, 4096),   # few tiles, deep K: split-K over 4 blocks
              (384, 512, 2080),    # split-K with a ragged last stage
              (100, 256, 520),     # partial M tile
              (256, 96, 64)]       # K too shallow to split


@pytest.mark.parametrize("m,n,k", TMA_SHAPES)
def test_gemm_nt_tma_split(m, n, k):
    """TMA-fed kernel incl. the split-K path: parity with float64 and bitwise
    reproducibility (the partial tiles are summed in split order)."""
    rng = np.random.default_rng(m + 5 * n + 11 * k)
    a = rng.uniform(-1, 1, size=(m, k))
    b = rng.uniform(-1, 1, size=(n, k))
    ta = torch.tensor(a, dtype=torch.float32, device="cuda")
    tb = torch.tensor(b, dtype=torch.float32, device="cuda")
    tbl = tb - (tb.view(torch.int32) & ~0x1FFF).view(torch.float32)
    outs = []
    for _ in range(3):
        tc = torch.full((m, n), float("nan"), device="cuda")
        _lib.check(_lib.lib().rgb_gemm_nt_tma(ctypes.c_void_p(ta.data_ptr()), ctypes.c_void_p(tb.data_ptr()),
                                              ctypes.c_void_p(tbl.data_ptr()), ctypes.c_void_p(tc.data_ptr()),
                                              m, n, k, _stream()))
        outs.append(tc.cpu().numpy())
    ref = a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T
    assert normwise(outs[0], ref) < 1e-5
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


MODES = [(1, 1, 1), (0, 1, 1), (1, 0, 1), (0, 0, 0)]  # (pairs, persistent, cluster split-K)


def _set_modes(mode):
    _lib.check(_lib.lib().rgb_set_tc_config(*mode))


@pytest.fixture()
def restore_tc_modes():
    yield
    _set_modes((1, 1, 1))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("m,n,k", [(8192, 2048, 256), (4096, 1000, 512), (600, 3000, 96)])
def test_gemm_nt_tma_kernel_variants(m, n, k, mode, restore_tc_modes):
    """CTA-pair, persistent (>= 2 waves) and plain kernels on the same products."""
    _set_modes(mode)
    rng = np.random.default_rng(m + n + k)
    a = rng.uniform(-1, 1, size=(m, k))
    b = rng.uniform(-1, 1, size=(n, k))
    ta = torch.tensor(a, dtype=torch.float32, device="cuda")
    tb = torch.tensor(b, dtype=torch.float32, device="cuda")
    tc = torch.full((m, n), float("nan"), device="cuda")
    _lib.check(_lib.lib().rgb_gemm_nt_tma(ctypes.c_void_p(ta.data_ptr()), ctypes.c_void_p(tb.data_ptr()),
                                          ctypes.c_void_p(tb.data_ptr()), ctypes.c_void_p(tc.data_ptr()),
                                          m, n, k, _stream()))
    ref = a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T
    assert normwise(tc.cpu().numpy(), ref) < 1e-5


@pytest.mark.parametrize("mode", [(1, 1, 1), (0, 1, 1)])
@pytest.mark.parametrize("m,n,k", [(8192, 3072, 1024), (16384, 1000, 512), (16384, 1024, 4096)])
def test_gemm_nt_persistent_tail_split(m, n, k, mode, restore_tc_modes):
    """Persistent launches whose last wave runs as column-half tiles
    (launch_persistent's tail split: 384 / 256 pair tiles on 74 pairs, 512
    single tiles on 148 SMs), ragged N included, deep K (chunked accumulation
    across the halves); every output element written (NaN-initialised)."""
    _set_modes(mode)
    rng = np.random.default_rng(m + n + k + 7)
    a = rng.uniform(-1, 1, size=(m, k))
    b = rng.uniform(-1, 1, size=(n, k))
    ta = torch.tensor(a, dtype=torch.float32, device="cuda")
    tb = torch.tensor(b, dtype=torch.float32, device="cuda")
    tc = torch.full((m, n), float("nan"), device="cuda")
    _lib.check(_lib.lib().rgb_gemm_nt_tma(ctypes.c_void_p(ta.data_ptr()), ctypes.c_void_p(tb.data_ptr()),
                                          ctypes.c_void_p(tb.data_ptr()), ctypes.c_void_p(tc.data_ptr()),
                                          m, n, k, _stream()))
    out = tc.cpu().numpy()
    assert not np.isnan(out).any()
    ref = a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T
    assert normwise(out, ref) < 1e-5


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("m,n,k", [(4096, 4096, 512), (1024, 1024, 2080), (96, 160, 333)])
def test_gemm_dw_tma(m, n, k, mode, restore_tc_modes):
    """TMA-fed dW (3-D MN-major maps): pairs, persistent and plain; ragged K."""
    _set_modes(mode)
    rng = np.random.default_rng(m * 3 + n + k)
    e = rng.uniform(-1, 1, size=(k, m))
    y = rng.uniform(-1, 1, size=(k, n))
    te = torch.tensor(e, dtype=torch.float32, device="cuda")
    ty = torch.tensor(y, dtype=torch.float32, device="cuda")
    tg = torch.full((m, n), float("nan"), device="cuda")
    _lib.check(_lib.lib().rgb_gemm_dw(ctypes.c_void_p(te.data_ptr()), ctypes.c_void_p(ty.data_ptr()),
                                      ctypes.c_void_p(tg.data_ptr()), m, n, k, ctypes.c_float(-1.0), 3,
                                      _stream()))
    ref = -(e.astype(np.float32).astype(np.float64).T @ y.astype(np.float32).astype(np.float64))
    # fp32 accumulation over K: the max-norm error's tail grows ~sqrt(K)
    assert normwise(tg.cpu().numpy(), ref) < 1e-5 * max(1.0, (k / 512) ** 0.5)


def test_engine_kernel_variants_agree(restore_tc_modes):
    """A cfg4-like step big enough for the persistent kernels and CTA pairs:
    outputs and weight gradients agree across the kernel variants (fp32
    summation order only), and the variant-free run matches the oracle on a
    smaller scale elsewhere."""
    net = P.build_stacked_lstm(1024, [1024, 1024], 1024)
    S, h, hp = 256, 32, 16
    rng = np.random.default_rng(5)
    xs = [rng.uniform(-1, 1, size=(hp * S, 1024)).astype(np.float32) for _ in range(3)]
    ts = [rng.integers(0, 1024, size=hp * S) for _ in range(3)]
    results = []
    for mode in [(1, 1, 1), (0, 0, 0)]:
        _set_modes(mode)
        w = P.Weights.init(net, 0)
        tr = P.Trainer(net, w, S, P.TrainConfig(h=h, h_prime=hp, lr=1e-3, iterations=1))
        for x, t in zip(xs, ts):
            tr.step(torch.tensor(x, device="cuda"), torch.tensor(t, device="cuda"))
        out = tr.state.read_y(net.output_layers()[0].id, tr.state.cursor - hp + 1, tr.state.cursor).cpu().numpy()
        results.append((out, tr.grads.flat.cpu().numpy(), w.flat[: w.n_params].cpu().numpy()))
    for a, b in zip(results[0], results[1]):
        assert normwise(a, b.astype(np.float64)) < 5e-5


def test_pair_cluster_split_k_opt_in():
    """CTA pairs combined with cluster split-K (opt-in variant, RGB_TC_PAIRSPLIT=1)
    computed in a subprocess so the environment switch takes effect."""
    import os
    import subprocess
    import sys
    code = (
        "import ctypes, numpy as np, torch\n"
        "from paper_1503_02852_b200 import _lib\n"
        "L = _lib.lib()\n"
        "rng = np.random.default_rng(3)\n"
        "m, n, k = 512, 2048, 1024\n"
        "a = rng.uniform(-1, 1, size=(m, k)); b = rng.uniform(-1, 1, size=(n, k))\n"
        "ta = torch.tensor(a, dtype=torch.float32, device='cuda'); tb = torch.tensor(b, dtype=torch.float32, device='cuda')\n"
        "tc = torch.full((m, n), float('nan'), device='cuda')\n"
        "P = lambda t: ctypes.c_void_p(t.data_ptr())\n"
        "_lib.check(L.rgb_gemm_nt_tma(P(ta), P(tb), P(tb), P(tc), m, n, k, ctypes.c_void_p(0)))\n"
        "torch.cuda.synchronize()\n"
        "ref = a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T\n"
        "err = np.abs(tc.cpu().numpy() - ref).max() / np.abs(ref).max()\n"
        "assert err < 1e-5, err\n"
        "print('ok', err)\n")
    env = dict(os.environ, RGB_TC_PAIRSPLIT="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]



def test_id_inputs_with_tensor_cores_forced():
    """Token-id gathers / sorted-scatter dW combined with tcgen05 GEMMs everywhere else."""
    from test_gpu_engine import run_pair
    L = _lib.lib()
    _lib.check(L.rgb_set_gemm_mode(2))
    try:
        assert run_pair(P.build_lstm(300, 32, 16), 3, 8, 4, 3, 0.05, 21, ids=True) < 1e-4
    finally:
        _lib.check(L.rgb_set_gemm_mode(0))


@pytest.mark.parametrize("kind", ["random", "coherent"])
@pytest.mark.parametrize("k", [4096, 16384])
def test_deep_k_accumulation_stays_fp32_exact(kind, k):
    """tcgen05 accumulates with truncation, so one accumulator's error grows
    with K (tools/accum_probe.py measured 3.1e-4 at K = 16384 before the
    K-chunked accumulation); the dW depth of cfg4 is h*S = 16384.  Both forms
    stay at the fp32 level (SIMT measured 6e-6 .. 7e-6 here)."""
    rng = np.random.default_rng(k)
    lo = 0.0 if kind == "coherent" else -1.0
    m = n = 512
    e, y = rng.uniform(lo, 1, size=(k, m)).astype(np.float32), rng.uniform(lo, 1, size=(k, n)).astype(np.float32)
    ref = e.astype(np.float64).T @ y.astype(np.float64)
    te, ty = torch.tensor(e, device="cuda"), torch.tensor(y, device="cuda")
    g = torch.empty((m, n), device="cuda")
    _lib.check(_lib.lib().rgb_gemm_dw(ctypes.c_void_p(te.data_ptr()), ctypes.c_void_p(ty.data_ptr()),
                                      ctypes.c_void_p(g.data_ptr()), m, n, k, ctypes.c_float(1.0), 3, _stream()))
    assert normwise(g.cpu().numpy(), ref) < 3e-5
    a, b = torch.tensor(np.ascontiguousarray(e.T), device="cuda"), torch.tensor(np.ascontiguousarray(y.T), device="cuda")
    c = torch.empty((m, n), device="cuda")
    _lib.check(_lib.lib().rgb_gemm_nt_tma(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                          ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(c.data_ptr()), m, n, k,
                                          _stream()))
    assert normwise(c.cpu().numpy(), ref) < 3e-5


# ---- plain-TF32 tensor-core mode (rgb_set_tc_precision(1)) ------------------
# The north_star allows a TF32 GEMM mode "to a separately stated bound".  One
# tcgen05 kind::tf32 product per k-step on operands rounded to nearest tf32
# (cvt.rna in the converter warps; the MMA alone would truncate, a biased
# 2^-11 relative error per operand); for U(-1,1) operands the normwise GEMM
# error is ~2e-4.  Stated bounds: GEMM and full training step
# (outputs, every delta / eps, weight gradients, weights after SGD) 2e-3
# normwise, loss 1e-2 relative.
TF32_GEMM_BOUND = 2e-3
TF32_STEP_BOUND = 2e-3


@pytest.fixture
def _tf32():
    L = _lib.lib()
    _lib.check(L.rgb_set_tc_precision(1))
    try:
        yield L
    finally:
        _lib.check(L.rgb_set_tc_precision(3))


def test_tc_precision_rejects_bad_values():
    L = _lib.lib()
    assert L.rgb_set_tc_precision(2) == _lib.RGB_ERR_KERNEL
    assert L.rgb_set_tc_precision(0) == _lib.RGB_ERR_KERNEL
    with pytest.raises(ValueError):
        P.set_tc_precision("bf16")
    P.set_tc_precision("tf32")
    P.set_tc_precision("3xtf32")


@pytest.mark.parametrize("m,n,k", [(256, 512, 1024), (1024, 2048, 1024), (200, 300, 70),
                                   # > 148 tiles (persistent kernels) and K deep enough to wrap the
                                   # 8- / 16-slot logical stage rings several times
                                   (4096, 4096, 2048)])
def test_gemm_tf32_mode(_tf32, m, n, k):
    """Both tcgen05 forms (NT and dW, incl. the TMA-fed dW) in plain TF32:
    inside the stated bound, and measurably less exact than 3xTF32 (the mode
    switch is real)."""
    rng = np.random.default_rng(m + 5 * n + k)
    a, b = rng.uniform(-1, 1, size=(m, k)), rng.uniform(-1, 1, size=(n, k))
    ta = torch.tensor(a, dtype=torch.float32, device="cuda")
    tb = torch.tensor(b, dtype=torch.float32, device="cuda")
    tc = torch.full((m, n), float("nan"), device="cuda")
    _lib.check(_tf32.rgb_gemm_nt(ctypes.c_void_p(ta.data_ptr()), ctypes.c_void_p(tb.data_ptr()),
                                 ctypes.c_void_p(tc.data_ptr()), m, n, k, 2, _stream()))
    ref = a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T
    err = normwise(tc.cpu().numpy(), ref)
    assert 1e-5 < err < TF32_GEMM_BOUND, err
    e, y = rng.uniform(-1, 1, size=(k, m)), rng.uniform(-1, 1, size=(k, n))
    te = torch.tensor(e, dtype=torch.float32, device="cuda")
    ty = torch.tensor(y, dtype=torch.float32, device="cuda")
    ref = -(e.astype(np.float32).astype(np.float64).T @ y.astype(np.float32).astype(np.float64))
    for mode in ([2, 3] if m % 32 == 0 and n % 32 == 0 else [2]):
        tg = torch.full((m, n), float("nan"), device="cuda")
        _lib.check(_tf32.rgb_gemm_dw(ctypes.c_void_p(te.data_ptr()), ctypes.c_void_p(ty.data_ptr()),
                                     ctypes.c_void_p(tg.data_ptr()), m, n, k, ctypes.c_float(-1.0), mode, _stream()))
        err = normwise(tg.cpu().numpy(), ref)
        assert 1e-5 < err < TF32_GEMM_BOUND, (mode, err)


def test_engine_parity_tf32_mode(_tf32):
    """Whole training steps with every GEMM on tcgen05 in plain TF32 against
    the float64 oracle, at the TF32 bound."""
    from test_gpu_engine import run_pair
    _lib.check(_tf32.rgb_set_gemm_mode(2))
    try:
        assert run_pair(P.build_lstm(39, 128, 39), 2, 32, 16, 3, 1e-3, 0, loss_tol=1e-2) < TF32_STEP_BOUND
        assert run_pair(P.build_stacked_lstm(256, [256, 256], 256), 64, 8, 4, 2, 1e-3, 4,
                        loss_tol=1e-2) < TF32_STEP_BOUND
    finally:
        _lib.check(_tf32.rgb_set_gemm_mode(0))


def test_cfg4_shape_tf32_mode(_tf32):
    """The cfg4 layer shapes (1024 wide, 2 layers, S = 256: persistent hoisted /
    dW kernels, per-frame launches) in plain TF32 against the oracle, at the
    TF32 bound, with every delta / eps compared."""
    from test_gpu_engine import run_pair
    worst = run_pair(P.build_stacked_lstm(1024, [1024, 1024], 1024), 256, 32, 16, 3, 1e-3, 6, loss_tol=1e-2)
    print(f"cfg4-shape TF32 step error {worst:.2e}")
    assert worst < TF32_STEP_BOUND


@pytest.mark.parametrize("S,frame_loop", [(256, 1), (256, 0)])
def test_persistent_frame_loop_matches_oracle(S, frame_loop):
    """The persistent tensor-core frame loop (rgb_set_frame_loop(1): one
    cooperative launch per recurrent loop, grid barrier per frame, split-K
    through DSMEM, the LSTM cell update fused into the epilogue) against the
    oracle, with every delta / eps / dW compared, and through CUDA-graph replay
    bit for bit equal to its eager steps."""
    from test_gpu_engine import run_pair
    L = _lib.lib()
    _lib.check(L.rgb_set_frame_loop(frame_loop))  # 0: the per-frame PDL launches of the same loops
    _lib.check(L.rgb_set_wavefront(0))  # (the wavefront runs frame loops per block, per-frame launches)
    n0 = ctypes.c_int64()
    _lib.check(L.rgb_launch_count(ctypes.byref(n0)))
    try:
        assert run_pair(P.build_stacked_lstm(256, [512, 512], 256), S, 16, 8, 3, 1e-3, 7) < 1e-4
        n1 = ctypes.c_int64()
        _lib.check(L.rgb_launch_count(ctypes.byref(n1)))
        # 3 iterations x (2 forward + 2 backward loops): the per-frame schedule
        # launches >= 8 + 16 kernels per loop pair; the frame loops keep it well below
        assert (n1.value - n0.value < 3 * 60) == bool(frame_loop)
        net = P.build_stacked_lstm(128, [512, 512], 128)
        cfg = P.TrainConfig(h=16, h_prime=8, lr=1e-4, iterations=1)  # raw gradient sums over S streams
        wa, wb = P.Weights.init(net, 2), P.Weights.init(net, 2)
        ta, tb = P.Trainer(net, wa, S, cfg), P.Trainer(net, wb, S, cfg)
        tb.enable_graphs()
        gx, gt = tb.graph_inputs()
        rng = np.random.default_rng(3)
        for _ in range(5):
            x = torch.tensor(rng.uniform(-1, 1, size=(8 * S, 128)), dtype=torch.float32, device="cuda")
            t = torch.tensor(rng.integers(0, 128, size=8 * S), device="cuda")
            ta.step(x, t)
            gx.copy_(x)
            gt.copy_(t)
            tb.step_graphed()
            assert ta.loss() == tb.loss()
        assert torch.equal(wa.flat, wb.flat)
    finally:
        _lib.check(L.rgb_set_frame_loop(1))
        _lib.check(L.rgb_set_wavefront(1))
