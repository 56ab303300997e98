"""The reference engine API over the sm_100a C ABI.

Same names, arguments, return types and guard errors as
``/root/reference/pkg/src/rnngraph/engine.py`` (``Weights``, ``GradStore``,
``BpttWindow``, ``StreamState``, ``forward_chunk``, ``inject_output_error``,
``loss_value``, ``backward_window``, ``sgd_update``, ``train_loop``), so a
caller of the reference switches by changing the import.  Arithmetic is fp32
on the device; tensors are torch CUDA tensors used purely as buffers (device
memory + the current stream).  Every numeric step is a kernel of
``librnngraph_b200.so`` -- there is no CPU or torch fallback: without the
library or an sm_100 device the calls raise.

Differences a caller can observe (all within the stated tolerance):

* values are float32 (the reference computes in float64);
* summation order differs (hoisted GEMMs, see schedule.py), so results are not
  bitwise equal to the reference but agree to <= 1e-4 normwise;
* ``Batch.values`` returned by this engine are CUDA tensors.
"""

from __future__ import annotations

import ctypes
import enum
import hashlib
import math
import struct
import time
from dataclasses import dataclass, field
from typing import Protocol

import numpy as np
import torch

from . import _lib
from .condense import CondensedGraph, condense
from .netdef import Activation, NetworkDef, Role, infer_shapes, save_network
from .schedule import EngineError, build_program, weight_offsets, weights_program

__all__ = [
    "Batch", "BpttWindow", "Criterion", "EngineError", "GradStore", "IterationMetrics", "StreamState",
    "TrainConfig", "Weights", "backward_window", "forward_chunk", "inject_output_error", "loss_value",
    "sgd_update", "train_loop",
]

DTYPE = torch.float32


class Criterion(enum.Enum):
    """(criterion, output activation) fused pairs (reference engine.py:94-104)."""

    CROSS_ENTROPY_SOFTMAX = "cross_entropy_softmax"
    MSE_IDENTITY = "mse_identity"


_CRIT_ACT = {Criterion.CROSS_ENTROPY_SOFTMAX: Activation.SOFTMAX, Criterion.MSE_IDENTITY: Activation.IDENTITY}
_CRIT_CODE = {Criterion.CROSS_ENTROPY_SOFTMAX: 0, Criterion.MSE_IDENTITY: 1}


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1503_02852_b200 needs a CUDA (sm_100) device; there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


class _Plan:
    """Owns one rgb_plan handle."""

    def __init__(self, words: np.ndarray):
        L = _lib.lib()
        self._lib = L
        words = np.ascontiguousarray(words, dtype=np.int32)
        h = ctypes.c_void_p()
        _lib.check(L.rgb_plan_create(words.ctypes.data_as(ctypes.c_void_p), words.size, ctypes.byref(h)),
                   "plan_create")
        self.handle = h

    def __del__(self):
        try:
            if self.handle:
                self._lib.rgb_plan_destroy(self.handle)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def workspace_bytes(self) -> int:
        v = ctypes.c_int64()
        _lib.check(self._lib.rgb_plan_workspace_bytes(self.handle, ctypes.byref(v)))
        return v.value

    @property
    def cursor(self) -> int:
        v = ctypes.c_int64()
        _lib.check(self._lib.rgb_plan_get_cursor(self.handle, ctypes.byref(v)))
        return v.value


# ---------------------------------------------------------------------------
# Batch (reference kernels.py:196-239)


@dataclass
class Batch:
    """``frames`` frames of ``streams`` streams, one sample per row,
    frame-major (row = t * streams + n).  ``values`` is a torch tensor (CUDA
    for this engine's outputs) or a numpy array (accepted as input)."""

    values: object
    frames: int
    streams: int

    def __post_init__(self):
        shape = tuple(self.values.shape)
        if len(shape) != 2 or shape[0] != self.frames * self.streams:
            raise _lib.KernelError(f"batch needs shape ({self.frames * self.streams}, width), got {shape}")

    @property
    def width(self) -> int:
        return int(self.values.shape[1])

    @classmethod
    def zeros(cls, width: int, frames: int, streams: int) -> "Batch":
        return cls(torch.zeros((frames * streams, width), dtype=DTYPE, device=_device()), frames, streams)

    def col(self, t: int, n: int):
        if not (0 <= t < self.frames and 0 <= n < self.streams):
            raise _lib.KernelError(f"sample ({t}, {n}) outside batch {self.frames}x{self.streams}")
        return self.values[t * self.streams + n]

    def frame(self, t: int):
        if not 0 <= t < self.frames:
            raise _lib.KernelError(f"frame {t} outside batch of {self.frames}")
        return self.values[t * self.streams:(t + 1) * self.streams]

    def stream(self, n: int):
        if not 0 <= n < self.streams:
            raise _lib.KernelError(f"stream {n} outside batch of {self.streams}")
        return self.values[n::self.streams]

    def copy(self) -> "Batch":
        v = self.values.clone() if isinstance(self.values, torch.Tensor) else self.values.copy()
        return Batch(v, self.frames, self.streams)

    def numpy(self) -> np.ndarray:
        v = self.values
        return v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v)


def _as_device_f32(values) -> torch.Tensor:
    if isinstance(values, torch.Tensor):
        t = values.to(device=_device(), dtype=DTYPE)
    else:
        t = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).to(_device())
    return t.contiguous()


# ---------------------------------------------------------------------------
# parameters (reference engine.py:111-162)


class Weights:
    """Dense connection matrices (dst, src) in one flat fp32 device buffer,
    plus the transposed copies used by the backward GEMMs (the reference's
    ``wt`` cache, refreshed after every update)."""

    def __init__(self, net: NetworkDef, w: dict | None = None, *, _flat=None, _flat_t=None):
        self.net = net
        self.offsets, self.n_params = weight_offsets(net)
        dev = _device()
        # W and W^T: n_params floats each (the 3xTF32 tensor-core GEMMs form the
        # tf32 residuals of their operands in shared memory; no residual buffers)
        n2 = max(self.n_params, 4)
        self.flat = _flat if _flat is not None else torch.zeros(n2, dtype=DTYPE, device=dev)
        self.flat_t = _flat_t if _flat_t is not None else torch.zeros_like(self.flat)
        self._plan = _Plan(weights_program(net))
        self.w, self.wt = {}, {}
        for c in net.iter_dense():
            r, k = net.layer(c.dst).size, net.layer(c.src).size
            o = self.offsets[c.id]
            self.w[c.id] = self.flat[o:o + r * k].view(r, k)
            self.wt[c.id] = self.flat_t[o:o + r * k].view(k, r)
        if w is not None:
            for cid, m in w.items():
                self.w[cid].copy_(torch.as_tensor(np.asarray(m) if not isinstance(m, torch.Tensor) else m,
                                                  dtype=DTYPE))
        if _flat_t is None:
            self.refresh()

    @classmethod
    def init(cls, net: NetworkDef, seed: int) -> "Weights":
        """U(-r, r), r = 1/sqrt(src_size), one PCG64 stream over connections in
        ascending id -- the reference's draw sequence (engine.py:126-136),
        drawn in float64 on the host and rounded to fp32."""
        shapes = infer_shapes(net)
        rng = np.random.default_rng(seed)
        w = {}
        for c in net.iter_dense():
            rows, cols = shapes[c.id]
            r = 1.0 / math.sqrt(cols)
            w[c.id] = rng.uniform(-r, r, size=(rows, cols))
        return cls(net, w)

    def refresh(self) -> None:
        _lib.check(_lib.lib().rgb_refresh_transpose(self._plan.handle, _ptr(self.flat), _ptr(self.flat_t), _stream()))

    def copy(self) -> "Weights":
        return Weights(self.net, _flat=self.flat.clone(), _flat_t=self.flat_t.clone())

    def numpy(self) -> dict[int, np.ndarray]:
        host = self.flat.detach().cpu().numpy().astype(np.float64)
        out = {}
        for c in self.net.iter_dense():
            r, k = self.net.layer(c.dst).size, self.net.layer(c.src).size
            o = self.offsets[c.id]
            out[c.id] = host[o:o + r * k].reshape(r, k)
        return out


@dataclass
class GradStore:
    """Loss gradient dE/dW per dense connection (flat fp32 device buffer with
    per-id views) and the number of (frame, stream) samples that contributed."""

    g: dict
    frames_streams: int = 0
    flat: torch.Tensor | None = None

    @classmethod
    def zeros(cls, net: NetworkDef) -> "GradStore":
        offsets, n = weight_offsets(net)
        flat = torch.zeros(max(n, 4), dtype=DTYPE, device=_device())
        g = {}
        for c in net.iter_dense():
            r, k = net.layer(c.dst).size, net.layer(c.src).size
            g[c.id] = flat[offsets[c.id]:offsets[c.id] + r * k].view(r, k)
        return cls(g=g, flat=flat)

    def add_(self, other: "GradStore") -> "GradStore":
        self.flat += other.flat  # plumbing: accumulate two gradient buffers
        self.frames_streams += other.frames_streams
        return self

    def numpy(self) -> dict[int, np.ndarray]:
        return {cid: m.detach().cpu().numpy().astype(np.float64) for cid, m in self.g.items()}


# ---------------------------------------------------------------------------
# window and state (reference engine.py:169-286)


@dataclass(frozen=True)
class BpttWindow:
    """Errors injected on (t1-h', t1], backpropagated through (t0', t1],
    t0' = max(t1-h, 0)."""

    t1: int
    h: int
    h_prime: int

    def __post_init__(self):
        if not 1 <= self.h_prime <= self.h:
            raise EngineError(f"need 1 <= h'={self.h_prime} <= h={self.h}")
        if self.t1 < self.h_prime:
            raise EngineError(f"t1={self.t1} leaves no room for {self.h_prime} injected frames")

    @property
    def t0(self) -> int:
        return self.t1 - self.h_prime

    @property
    def t0_prime(self) -> int:
        return max(self.t1 - self.h, 0)

    @property
    def frames(self) -> int:
        return self.t1 - self.t0_prime


_PROGRAMS: dict = {}


def _program(net: NetworkDef, S: int, h: int, chunk: int | None):
    key = (net, S, h, chunk)
    if key not in _PROGRAMS:
        _PROGRAMS[key] = build_program(net, condense(net), S, h, chunk)
    return _PROGRAMS[key]


class StreamState:
    """Activation history of ``n_streams`` parallel streams on the device.

    Per layer a mirrored ring of 2*cap frames (cap >= h + max_delay) holds the
    newest frames, frame-major, so frames t <= 0 read as zeros and advancing
    is free (no memmove).  ``chunk`` (the usual h') rounds cap up to a multiple
    of it.  Guards and addressing match the reference (engine.py:197-286).
    """

    def __init__(self, net: NetworkDef, n_streams: int, h: int, *, chunk: int | None = None):
        if n_streams < 1 or h < 1:
            raise EngineError(f"need n_streams >= 1 and h >= 1, got {n_streams}, {h}")
        self.net, self.n, self.h = net, n_streams, h
        self.capacity = h + net.max_delay
        self.program = _program(net, n_streams, h, chunk)
        self._plan = _Plan(self.program.words)
        nbytes = self._plan.workspace_bytes()
        self.workspace = torch.zeros(max(nbytes // 4, 4), dtype=DTYPE, device=_device())
        _lib.check(_lib.lib().rgb_plan_bind(self._plan.handle, _ptr(self.workspace)))
        self.input_mode: str | None = None

    @property
    def cursor(self) -> int:
        return self._plan.cursor

    @property
    def base(self) -> int:
        return self.cursor - self.capacity

    def rows(self, t_lo: int, t_hi: int) -> slice:
        """Row slice of frames t_lo..t_hi inside the (virtual) reference layout."""
        if t_lo <= self.base or t_hi > self.cursor:
            raise EngineError(f"frames [{t_lo}, {t_hi}] outside resident window ({self.base}, {self.cursor}]")
        return slice((t_lo - self.base - 1) * self.n, (t_hi - self.base) * self.n)

    def _ring(self, buf: int, t_lo: int, t_hi: int) -> torch.Tensor:
        self.rows(t_lo, t_hi)  # guard
        L = self.program.layout
        kind, width, off, _ = L.bufs[buf]
        slot = t_lo % L.cap
        fr = self.n * width
        start = off + slot * fr
        return self.workspace[start:start + (t_hi - t_lo + 1) * fr].view(-1, width)

    def read_y(self, layer_id: int, t_lo: int, t_hi: int) -> torch.Tensor:
        """Activation rows for frames t_lo..t_hi (device view; do not mutate)."""
        return self._ring(self.program.y_buf[layer_id], t_lo, t_hi)

    def reset_stream(self, n: int) -> None:
        """Zero one stream's history (sequence boundary, engine.py:267-276)."""
        if not 0 <= n < self.n:
            raise EngineError(f"stream {n} outside [0, {self.n})")
        _lib.check(_lib.lib().rgb_reset_stream(self._plan.handle, n, _stream()))

    def copy(self) -> "StreamState":
        dup = StreamState.__new__(StreamState)
        dup.net, dup.n, dup.h, dup.capacity = self.net, self.n, self.h, self.capacity
        dup.program = self.program
        dup._plan = _Plan(self.program.words)
        dup.workspace = self.workspace.clone()
        _lib.check(_lib.lib().rgb_plan_bind(dup._plan.handle, _ptr(dup.workspace)))
        _lib.check(_lib.lib().rgb_plan_set_cursor(dup._plan.handle, self.cursor))
        dup.input_mode = self.input_mode
        return dup


def _single_io(net: NetworkDef):
    ins, outs = net.input_layers(), net.output_layers()
    if len(ins) != 1 or len(outs) != 1:
        raise EngineError(f"engine supports exactly one input and one output layer, got {len(ins)} and {len(outs)}")
    return ins[0], outs[0]


# ---------------------------------------------------------------------------
# forward (reference engine.py:352-418)


def _input_rows(lin, state: StreamState, inputs):
    """Validate a chunk and return (device fp32 rows or int64 ids, frames, mode)."""
    if isinstance(inputs, Batch):
        if inputs.streams != state.n:
            raise EngineError(f"chunk has {inputs.streams} streams, state has {state.n}")
        if inputs.width != lin.size:
            raise EngineError(f"input width {inputs.width} != layer size {lin.size}")
        return _as_device_f32(inputs.values), inputs.frames, "dense"
    ids = inputs if isinstance(inputs, torch.Tensor) else np.asarray(inputs)
    kind = ids.dtype.is_floating_point if isinstance(ids, torch.Tensor) else ids.dtype.kind not in "iu"
    if kind or ids.ndim != 1:
        raise EngineError("id inputs must be a 1-d integer array")
    if ids.shape[0] % state.n:
        raise EngineError(f"{ids.shape[0]} ids do not tile {state.n} streams")
    frames = ids.shape[0] // state.n
    if ids.shape[0] and (int(ids.min()) < 0 or int(ids.max()) >= lin.size):
        raise EngineError(f"input ids outside [0, {lin.size})")
    for c in state.net.posterior(lin.id):
        if state.net.connection(c).weight_kind.value != "dense":
            raise EngineError(f"connection {c}: identity weight from an id-driven input layer is not supported")
    # the device keeps an id history: no one-hot rows (W^T row gathers forward,
    # sorted scatter for dW -- rgb_forward_chunk_ids)
    return torch.as_tensor(ids, dtype=torch.int64).to(_device()).contiguous(), frames, "ids"


def forward_chunk(net: NetworkDef, cg: CondensedGraph, weights: Weights, state: StreamState, inputs, *,
                  frame_parallel: bool = True, check_finite: bool = False) -> Batch:
    """Advance all streams by one chunk; return the output activations.

    ``inputs``: a dense Batch (numpy or torch values) or an int64 id array
    (one-hot rows).  ``frame_parallel=False`` runs the frame-by-frame
    baseline schedule."""
    lin, lout = _single_io(net)
    x, frames, mode = _input_rows(lin, state, inputs)
    if state.input_mode is None:
        state.input_mode = mode
    elif state.input_mode != mode:
        raise EngineError(f"chunk mode {mode!r} != stream mode {state.input_mode!r}")
    if frames < 1:
        raise EngineError("empty chunk")
    if frames > state.h:
        raise EngineError(f"advance by {frames} outside [1, h={state.h}]")
    L = _lib.lib()
    if mode == "ids":
        _lib.check(L.rgb_forward_chunk_ids(state._plan.handle, _ptr(weights.flat), _ptr(weights.flat_t), _ptr(x), 0,
                                           frames, 0 if frame_parallel else 1, _stream()), "forward_chunk")
    else:
        _lib.check(L.rgb_forward_chunk(state._plan.handle, _ptr(weights.flat), _ptr(x), 0, frames,
                                       0 if frame_parallel else 1, _stream()), "forward_chunk")
    t_hi = state.cursor
    t_lo = t_hi - frames + 1
    if check_finite:
        for l in net.layers:
            bad = ctypes.c_int64()
            _lib.check(L.rgb_count_nonfinite(state._plan.handle, state.program.y_buf[l.id], t_lo, t_hi,
                                             ctypes.byref(bad), _stream()))
            if bad.value:
                raise FloatingPointError(f"{bad.value} non-finite values in activations of layer {l.name!r}")
    return Batch(state.read_y(lout.id, t_lo, t_hi).clone(), frames, state.n)


# ---------------------------------------------------------------------------
# error injection and loss (reference engine.py:425-474)


def _target_arg(target, rows: int, width: int):
    """(device tensor, kind) for a Batch / id array target."""
    if isinstance(target, Batch):
        return _as_device_f32(target.values), 2
    ids = torch.as_tensor(target if isinstance(target, torch.Tensor) else np.asarray(target))
    return ids.to(device=_device(), dtype=torch.int64).contiguous(), 0


def _inject(target, output: Batch, criterion: Criterion):
    rows, width = output.values.shape
    tgt, kind = _target_arg(target, rows, width)
    y = _as_device_f32(output.values)
    delta = torch.empty_like(y)
    scratch = torch.empty(rows + 1, dtype=torch.float64, device=_device())
    _lib.check(_lib.lib().rgb_inject_rows(_ptr(y), _ptr(tgt), kind, _CRIT_CODE[criterion], _ptr(delta),
                                          _ptr(scratch), ctypes.c_void_p(scratch.data_ptr() + 8 * rows),
                                          rows, width, _stream()))
    return delta, scratch[rows:]


def inject_output_error(target, output: Batch, criterion: Criterion, activation: Activation) -> Batch:
    """delta_out = d - y for the fused (criterion, activation) pairs."""
    want = _CRIT_ACT[criterion]
    if activation is not want:
        raise EngineError(f"{criterion.value} requires {want.value} output activation, got {activation.value}")
    if isinstance(target, Batch):
        if tuple(target.values.shape) != tuple(output.values.shape):
            raise EngineError(f"target shape {tuple(target.values.shape)} != output {tuple(output.values.shape)}")
    else:
        if criterion is not Criterion.CROSS_ENTROPY_SOFTMAX:
            raise EngineError("class-id targets are only defined for cross-entropy")
        n = len(target)
        if n != output.values.shape[0]:
            raise EngineError(f"need {output.values.shape[0]} target ids, got ({n},)")
    delta, _ = _inject(target, output, criterion)
    return Batch(delta, output.frames, output.streams)


def loss_value(target, output: Batch, criterion: Criterion) -> float:
    """Total (summed) loss over the batch, accumulated in fp64 on the device."""
    if criterion is Criterion.MSE_IDENTITY and not isinstance(target, Batch):
        raise EngineError("mean-squared error needs dense targets")
    _, loss = _inject(target, output, criterion)
    return float(loss.item())


# ---------------------------------------------------------------------------
# backward (reference engine.py:481-599)


def _view(state: StreamState, buf: int, t_lo: int, t_hi: int) -> torch.Tensor:
    """Device view of schedule buffer ``buf`` over frames [t_lo, t_hi] through
    rgb_window_view (rows frame-major, one row per stream)."""
    ptr, width = ctypes.c_void_p(), ctypes.c_int()
    _lib.check(_lib.lib().rgb_window_view(state._plan.handle, buf, t_lo, t_hi, ctypes.byref(ptr), ctypes.byref(width)),
               "window_view")
    off = (ptr.value - state.workspace.data_ptr()) // 4
    n = (t_hi - t_lo + 1) * state.n * width.value
    return state.workspace[off:off + n].view(-1, width.value)


def window_errors(state: StreamState, t1: int, h: int) -> tuple[dict, dict]:
    """(delta, eps) of the last backward window ending at t1: per-layer deltas
    and per-edge eps over frames (t0', t1], t0' = max(t1 - h, 0), as the
    reference computes them (engine.py:512-566; eps = delta of the destination
    for additive layers, delta times the other factors' z for multiplicative
    ones).  Device views, valid until the next backward_window."""
    net, L = state.net, state.program.layout
    t0p = max(t1 - h, 0)
    delta, eps = {}, {}
    if t1 <= t0p:
        return delta, eps
    for name, buf in L.names.items():
        if name.startswith("d") and name[1:].isdigit():
            delta[int(name[1:])] = _view(state, buf, t0p + 1, t1)
    for c in net.connections:
        if f"e{c.id}" in L.names:
            eps[c.id] = _view(state, L.names[f"e{c.id}"], t0p + 1, t1)
        elif c.dst in delta:
            eps[c.id] = delta[c.dst]
    return delta, eps


def backward_window(net: NetworkDef, cg: CondensedGraph, weights: Weights, state: StreamState, window: BpttWindow,
                    delta_out: Batch, *, frame_parallel: bool = True, capture: dict | None = None) -> GradStore:
    """Backpropagate the injected output errors through the window and return
    dE/dW.  Pure with respect to ``state``.  ``capture`` (a dict, optional;
    no reference counterpart) receives ``delta`` / ``eps`` per layer / edge id
    over (t0', t1] as device views (window_errors)."""
    _single_io(net)
    n = state.n
    if window.t1 != state.cursor:
        raise EngineError(f"window t1={window.t1} != stream cursor {state.cursor}")
    if window.h > state.h:
        raise EngineError(f"window h={window.h} exceeds state h={state.h}")
    if (delta_out.frames, delta_out.streams) != (window.h_prime, n):
        raise EngineError(f"delta_out is {delta_out.frames}x{delta_out.streams}, window wants {window.h_prime}x{n}")
    if state.program.softmax_feeds is not None:
        raise EngineError(f"softmax layer {state.program.softmax_feeds!r} feeds other layers; its derivative only "
                          "exists fused with cross-entropy injection")
    L = _lib.lib()
    d = _as_device_f32(delta_out.values)
    _lib.check(L.rgb_set_injection(state._plan.handle, _ptr(d), window.h_prime, _stream()))
    grads = GradStore.zeros(net)
    grads.frames_streams = window.frames * n
    _lib.check(L.rgb_backward_window(state._plan.handle, _ptr(weights.flat_t), _ptr(grads.flat), window.h,
                                     window.h_prime, 0 if frame_parallel else 1, _stream()), "backward_window")
    if capture is not None:
        capture["delta"], capture["eps"] = window_errors(state, window.t1, window.h)
    return grads


# ---------------------------------------------------------------------------
# update (reference engine.py:606-612)


def sgd_update(weights: Weights, grads: GradStore, lr: float) -> None:
    """W <- W - lr * grad, then refresh the transpose cache."""
    if not lr > 0.0:
        raise EngineError(f"learning rate must be positive, got {lr}")
    _lib.check(_lib.lib().rgb_sgd_update(weights._plan.handle, _ptr(weights.flat), _ptr(weights.flat_t),
                                         _ptr(grads.flat), ctypes.c_float(lr), _stream()))


# ---------------------------------------------------------------------------
# checkpoints (reference engine.py:615-665; same RNNG v1 byte format, so files
# move between the two implementations)


_TC_TERMS = {"3xtf32": 3, "tf32": 1}


def set_tc_precision(mode: str) -> None:
    """Tensor-core GEMM precision for subsequently launched (and captured)
    steps: ``"3xtf32"`` (default, fp32-exact) or ``"tf32"`` (the separately
    bounded mode: 2e-2 normwise per training step, tests/test_gpu_gemm.py).
    No reference counterpart -- the reference computes in float64
    (kernels.py:84-103).  CUDA graphs captured earlier keep their mode."""
    if mode not in _TC_TERMS:
        raise ValueError(f"tensor-core precision must be one of {sorted(_TC_TERMS)}, got {mode!r}")
    _lib.check(_lib.lib().rgb_set_tc_precision(_TC_TERMS[mode]))


class CheckpointError(EngineError):
    """Mirror of the reference ``CheckpointError`` (engine.py:90)."""


_CKPT_MAGIC = b"RNNG"
_CKPT_VERSION = 1


def structure_hash(net: NetworkDef) -> bytes:
    """First 8 bytes of SHA-256 over the canonical network document."""
    return hashlib.sha256(save_network(net).encode()).digest()[:8]


def save_checkpoint(path: str, net: NetworkDef, weights: Weights) -> None:
    """Header (magic, version, structure hash, count) then, per dense
    connection in ascending id, (id, rows, cols) and the matrix as
    little-endian float64 (fp32 values widen exactly)."""
    mats = weights.numpy()
    parts = [_CKPT_MAGIC, struct.pack("<I", _CKPT_VERSION), structure_hash(net), struct.pack("<I", len(mats))]
    for cid in sorted(mats):
        m = np.asarray(mats[cid], dtype="<f8")
        parts.append(struct.pack("<III", cid, m.shape[0], m.shape[1]))
        parts.append(np.ascontiguousarray(m).tobytes())
    with open(path, "wb") as fh:
        fh.write(b"".join(parts))


def load_checkpoint(path: str, net: NetworkDef) -> Weights:
    """Read an RNNG v1 file into device weights (float64 -> fp32)."""
    return Weights(net, read_checkpoint(path, net))


def read_checkpoint(path: str, net: NetworkDef) -> dict:
    """Parse and validate an RNNG v1 file: {connection id: float64 matrix}."""
    with open(path, "rb") as fh:
        blob = fh.read()
    pos = 0

    def take(n: int) -> bytes:
        nonlocal pos
        if pos + n > len(blob):
            raise CheckpointError(f"{path}: truncated checkpoint")
        out = blob[pos:pos + n]
        pos += n
        return out

    if take(4) != _CKPT_MAGIC:
        raise CheckpointError(f"{path}: not a checkpoint file")
    (version,) = struct.unpack("<I", take(4))
    if version != _CKPT_VERSION:
        raise CheckpointError(f"{path}: unsupported version {version}")
    if take(8) != structure_hash(net):
        raise CheckpointError(f"{path}: checkpoint belongs to a different network structure")
    shapes = infer_shapes(net)
    (count,) = struct.unpack("<I", take(4))
    mats: dict[int, np.ndarray] = {}
    for _ in range(count):
        cid, rows, cols = struct.unpack("<III", take(12))
        if shapes.get(cid) != (rows, cols):
            raise CheckpointError(f"{path}: connection {cid} has shape {(rows, cols)}")
        mats[cid] = np.frombuffer(take(rows * cols * 8), dtype="<f8").reshape(rows, cols).copy()
    want = {c.id for c in net.iter_dense()}
    if set(mats) != want:
        raise CheckpointError(f"{path}: connection ids {sorted(mats)} != network {sorted(want)}")
    return mats


# ---------------------------------------------------------------------------
# training (reference engine.py:672-762)


class StreamSource(Protocol):
    n_streams: int

    def next_batch(self, h_prime: int): ...


@dataclass
class TrainConfig:
    h: int
    h_prime: int
    lr: float
    iterations: int
    seed: int = 0
    criterion: Criterion = Criterion.CROSS_ENTROPY_SOFTMAX
    reset_on_sequence_boundary: bool = False
    frame_parallel: bool = True
    check_finite: bool = False
    log_every: int = 0

    def __post_init__(self):
        if not 1 <= self.h_prime <= self.h:
            raise EngineError(f"need 1 <= h'={self.h_prime} <= h={self.h}")
        if self.iterations < 1:
            raise EngineError("need at least one iteration")


@dataclass
class IterationMetrics:
    iteration: int
    loss: float
    frames: int
    seconds: float
    words_per_sec: float


class Trainer:
    """One BPTT(h; h') iteration as four C-ABI calls on the current stream:
    forward_chunk -> fused softmax-xent inject + loss -> backward_window ->
    SGD (+ W^T refresh).  ``step`` does not synchronise; ``loss`` does."""

    def __init__(self, net: NetworkDef, weights: Weights, n_streams: int, config: TrainConfig):
        _, self.lout = _single_io(net)
        want = _CRIT_ACT[config.criterion]
        if self.lout.activation is not want:
            raise EngineError(f"{config.criterion.value} requires {want.value} output, network has "
                              f"{self.lout.activation.value}")
        self.net, self.weights, self.cfg = net, weights, config
        self.state = StreamState(net, n_streams, config.h, chunk=config.h_prime)
        self.grads = GradStore.zeros(net)
        self._lib = _lib.lib()
        self._seq = 0 if config.frame_parallel else 1

    def step(self, inputs, targets, exchange=None) -> None:
        """One iteration.  ``exchange`` (dist.GradientExchange) sums the
        gradient buffer over ranks between backward and SGD."""
        L, st, plan = self._lib, self._stream(), self.state._plan.handle
        hp = self.cfg.h_prime
        x, on_host, mode = self._check_inputs(inputs)
        targets = self._check_targets(targets)
        if mode == "ids":  # token ids: id history, W^T row gathers, sorted-scatter dW
            _lib.check(L.rgb_forward_chunk_ids(plan, _ptr(self.weights.flat), _ptr(self.weights.flat_t), _ptr(x),
                                               on_host, hp, self._seq, st))
        else:
            _lib.check(L.rgb_forward_chunk(plan, _ptr(self.weights.flat), _ptr(x), on_host, hp, self._seq, st))
        if self.cfg.check_finite:
            t_hi = self.state.cursor
            for l in self.net.layers:
                bad = ctypes.c_int64()
                _lib.check(L.rgb_count_nonfinite(plan, self.state.program.y_buf[l.id], t_hi - hp + 1, t_hi,
                                                 ctypes.byref(bad), st))
                if bad.value:
                    raise FloatingPointError(f"{bad.value} non-finite values in activations of layer {l.name!r}")
        tkind = 2 if targets.is_floating_point() else (0 if targets.dtype == torch.int64 else 1)
        _lib.check(L.rgb_inject_output_error(plan, _ptr(targets), tkind, 0 if targets.is_cuda else 1,
                                             _CRIT_CODE[self.cfg.criterion], hp, st))
        if self.state.program.softmax_feeds is not None:
            raise EngineError(f"softmax layer {self.state.program.softmax_feeds!r} feeds other layers")
        if exchange is not None and getattr(exchange, "bucketed", False) and not self._seq:
            # bucketed backward: each supernode's dW summed over the GPUs while
            # the backward below it runs (C ABI + NCCL, dist.NcclExchange)
            _lib.check(L.rgb_backward_window_allreduce(plan, _ptr(self.weights.flat_t), _ptr(self.grads.flat),
                                                       self.cfg.h, hp, exchange.handle, st))
        else:
            _lib.check(L.rgb_backward_window(plan, _ptr(self.weights.flat_t), _ptr(self.grads.flat), self.cfg.h, hp,
                                             self._seq, st))
            if exchange is not None:
                exchange.allreduce_(self.grads.flat)
        _lib.check(L.rgb_sgd_update(self.weights._plan.handle, _ptr(self.weights.flat), _ptr(self.weights.flat_t),
                                    _ptr(self.grads.flat), ctypes.c_float(self.cfg.lr), st))

    # ---- argument validation (reference forward_chunk / inject_output_error guards,
    # engine.py:372-403, 436-456): shape, dtype, frames == h', streams == S; id
    # ranges of host arrays here, of device tensors by the kernels' error flag
    # (reported by loss() / check_inputs() without a sync inside step)
    def _check_inputs(self, inputs):
        S, hp = self.state.n, self.cfg.h_prime
        lin = self.net.layer(self.net.input_layers()[0].id)
        if not isinstance(inputs, torch.Tensor):
            x, frames, mode = _input_rows(lin, self.state, inputs)
            if frames != hp:
                raise EngineError(f"chunk has {frames} frames, step wants h'={hp}")
            return x, 0, mode
        if inputs.is_floating_point():
            if tuple(inputs.shape) != (hp * S, lin.size):
                raise EngineError(f"dense inputs must be ({hp * S}, {lin.size}) = (h'*S, n_in), got "
                                  f"{tuple(inputs.shape)}")
            x = inputs if inputs.dtype == DTYPE else inputs.to(DTYPE)
            return x.contiguous(), 0 if x.is_cuda else 1, "dense"
        if inputs.ndim != 1 or inputs.shape[0] != hp * S:
            raise EngineError(f"id inputs must be ({hp * S},) = (h'*S,), got {tuple(inputs.shape)}")
        if not inputs.is_cuda and inputs.numel() and (int(inputs.min()) < 0 or int(inputs.max()) >= lin.size):
            raise EngineError(f"input ids outside [0, {lin.size})")
        x = inputs if inputs.dtype == torch.int64 else inputs.to(torch.int64)
        return x.contiguous(), 0 if x.is_cuda else 1, "ids"

    def _check_targets(self, targets) -> torch.Tensor:
        S, hp = self.state.n, self.cfg.h_prime
        n_out = self.lout.size
        if isinstance(targets, Batch):
            targets = _as_device_f32(targets.values)
        elif not isinstance(targets, torch.Tensor):
            targets = torch.as_tensor(np.asarray(targets))
        if targets.is_floating_point():
            if tuple(targets.shape) != (hp * S, n_out):
                raise EngineError(f"dense targets must be ({hp * S}, {n_out}), got {tuple(targets.shape)}")
            return (targets if targets.dtype == DTYPE else targets.to(DTYPE)).contiguous()
        if self.cfg.criterion is not Criterion.CROSS_ENTROPY_SOFTMAX:
            raise EngineError("class-id targets are only defined for cross-entropy")
        if targets.ndim != 1 or targets.shape[0] != hp * S:
            raise EngineError(f"need {hp * S} target ids, got {tuple(targets.shape)}")
        if not targets.is_cuda and targets.numel() and (int(targets.min()) < 0 or int(targets.max()) >= n_out):
            raise IndexError(f"target ids outside [0, {n_out})")
        if targets.dtype not in (torch.int64, torch.int32):
            targets = targets.to(torch.int64)
        return targets.contiguous()

    def check_inputs(self) -> None:
        """Raise EngineError if a device-side id of an earlier step was out of
        range (synchronises)."""
        _lib.check(self._lib.rgb_check_inputs(self.state._plan.handle, self._stream()))

    def loss(self) -> float:
        v = ctypes.c_double()
        _lib.check(self._lib.rgb_read_loss(self.state._plan.handle, ctypes.byref(v), self._stream()))
        return v.value

    # ---- CUDA-graph replay of whole iterations --------------------------------
    def enable_graphs(self, exchange=None, ids: bool = False) -> None:
        """Capture the iteration once per ring phase and replay it.

        Every kernel argument of an iteration depends on the cursor only
        through (cursor mod ring capacity) and through differences of frame
        numbers, so an iteration captured at cursor c is valid at every cursor
        c + k*cap.  Inputs/targets come from static device buffers
        (``graph_inputs``); the loss stays on the device (``loss()`` syncs)."""
        hp = self.cfg.h_prime
        n_in = self.net.input_layers()[0].size
        dev = _device()
        S = self.state.n
        # ids=True: the graphs read token ids (int64) instead of dense rows
        self.gx = (torch.zeros((hp * S,), dtype=torch.int64, device=dev) if ids
                   else torch.zeros((hp * S, n_in), dtype=DTYPE, device=dev))
        self.gt = torch.zeros((hp * S,), dtype=torch.int64, device=dev)
        self._graphs = {}
        self._exchange = exchange
        self._cap = self.state.program.layout.cap
        # double-buffered staging of host inputs on a copy stream
        self._copy_stream = torch.cuda.Stream(device=dev)
        self._stage = [(torch.empty_like(self.gx), torch.empty_like(self.gt)) for _ in range(2)]
        self._stage_free = [torch.cuda.Event() for _ in range(2)]
        self._stage_ready = [torch.cuda.Event() for _ in range(2)]
        self._stage_next = 0
        self._staged = None
        self._loss_host = torch.zeros(2, dtype=torch.float64).pin_memory()
        self._loss_slot = 0

    def graph_inputs(self):
        """(x, targets) device buffers the next graphed step reads."""
        return self.gx, self.gt

    def stage_inputs(self, inputs: torch.Tensor, targets: torch.Tensor) -> None:
        """Start the host->device copy of the NEXT graphed iteration's inputs
        (pinned host tensors) on a copy stream, overlapping the running
        iteration; ``step_graphed`` consumes them."""
        k = self._stage_next
        sx, stt = self._stage[k]
        with torch.cuda.stream(self._copy_stream):
            self._copy_stream.wait_event(self._stage_free[k])  # previous consumer of this slot
            sx.copy_(inputs, non_blocking=True)
            stt.copy_(targets, non_blocking=True)
            self._stage_ready[k].record(self._copy_stream)
        self._staged = k
        self._stage_next = 1 - k

    def loss_async(self):
        """Enqueue the read-back of this iteration's loss; returns a callable
        that waits for it and returns the float."""
        slot = self._loss_slot
        self._loss_slot = 1 - slot
        dst = self._loss_host[slot:slot + 1]
        _lib.check(self._lib.rgb_read_loss_async(self.state._plan.handle, ctypes.c_void_p(dst.data_ptr()),
                                                 self._stream()))
        ev = torch.cuda.Event()
        ev.record()

        def wait() -> float:
            ev.synchronize()
            return float(dst[0])
        return wait

    def step_graphed(self) -> None:
        """One iteration on (graph_inputs()), replayed from a captured graph."""
        hp = self.cfg.h_prime
        if self._staged is not None:  # inputs staged by stage_inputs: device-to-device into the graph buffers
            k = self._staged
            cur = torch.cuda.current_stream()
            cur.wait_event(self._stage_ready[k])
            self.gx.copy_(self._stage[k][0], non_blocking=True)
            self.gt.copy_(self._stage[k][1], non_blocking=True)
            self._stage_free[k].record(cur)
            self._staged = None
        if not self._graphs and not getattr(self, "_graph_warm", False):
            # first call runs eagerly: it builds the tensor maps and SCC plans
            # (host-synchronous work that must not happen inside a capture)
            self.step(self.gx, self.gt, self._exchange)
            self._graph_warm = True
            return
        start = self.state.cursor
        g = self._graphs.get(start % self._cap)
        if g is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):  # records only; rewinds the host cursor below
                self.step(self.gx, self.gt, self._exchange)
            self._graphs[start % self._cap] = g
        g.replay()
        _lib.check(self._lib.rgb_plan_set_cursor(self.state._plan.handle, start + hp))

    @staticmethod
    def _stream():
        return _stream()


def train_loop(net: NetworkDef, streams: StreamSource, config: TrainConfig, weights: Weights | None = None,
               log=None) -> tuple[Weights, list[IterationMetrics]]:
    """SGD over BPTT(h; h') windows; every iteration consumes h' new frames
    per stream (minibatch h' * n_streams)."""
    condense(net)
    if weights is None:
        weights = Weights.init(net, config.seed)
    tr = Trainer(net, weights, streams.n_streams, config)
    metrics: list[IterationMetrics] = []
    for it in range(config.iterations):
        start = time.perf_counter()
        chunk = streams.next_batch(config.h_prime)
        if config.reset_on_sequence_boundary and getattr(chunk, "new_sequence", None) is not None:
            for s in np.flatnonzero(np.asarray(chunk.new_sequence)):
                tr.state.reset_stream(int(s))
        tr.step(chunk.inputs, chunk.targets)
        total = tr.loss()
        seconds = time.perf_counter() - start
        samples = config.h_prime * streams.n_streams
        m = IterationMetrics(it, total / samples, samples, seconds, samples / seconds if seconds > 0 else float("inf"))
        metrics.append(m)
        if log is not None and config.log_every and (it % config.log_every == 0 or it == config.iterations - 1):
            log(f"iter {it:5d}  loss {m.loss:.6f}  {m.words_per_sec:,.0f} words/s")
    return weights, metrics
