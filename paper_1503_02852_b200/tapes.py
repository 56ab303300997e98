"""Device-fed token tapes: the reference's StreamTape / StreamSet /
make_streams (data.py:117-207) with the corpus resident on the GPU.

Per chunk, the host advances each stream's tape arithmetically -- one step
per document span, not per token -- and emits the corpus position of every
input and look-ahead target token; one kernel (rgb_tape_gather) gathers the
ids into frame-major device buffers.  The token sequence is identical to the
reference's for the same corpus and seed (same dealing, same per-tape
reshuffles at epoch ends), so train_loop sees the same data either way.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass
class DeviceChunk:
    inputs: torch.Tensor        # (h' * N,) int64 on the device, frame-major
    targets: torch.Tensor       # (h' * N,) int64 on the device
    new_sequence: np.ndarray    # (N,) bool: the stream starts a fresh document


class _TapeCursor:
    """Host bookkeeping of one tape (reference StreamTape, data.py:117-155)."""

    def __init__(self, lengths: np.ndarray, starts: np.ndarray, seed: int):
        self.len = lengths
        self.start = starts
        self.rng = np.random.default_rng(seed)
        self.order = list(range(len(lengths)))
        self.at = 0
        self.off = 0

    def _advance(self, n: int, out: list) -> None:
        """Consume n tokens, appending (corpus position, count) spans."""
        while n > 0:
            d = self.order[self.at]
            take = min(n, int(self.len[d]) - self.off)
            out.append((int(self.start[d]) + self.off, take))
            self.off += take
            n -= take
            if self.off >= self.len[d]:
                self.at += 1
                self.off = 0
                if self.at >= len(self.order):
                    self.rng.shuffle(self.order)  # same draw as the reference tape
                    self.at = 0

    def read(self, k: int) -> tuple[np.ndarray, bool]:
        """Positions of k inputs followed by the look-ahead token."""
        boundary = self.off == 0
        spans: list = []
        self._advance(k, spans)
        d = self.order[self.at]  # peek the next token without consuming it
        spans.append((int(self.start[d]) + self.off, 1))
        pos = np.concatenate([np.arange(p, p + c, dtype=np.int64) for p, c in spans])
        return pos, boundary


class TapePlanner:
    """Host side of the device tapes: the reference's dealing of documents to
    N tapes (make_streams, data.py:183-207) and each tape's cursor."""

    def __init__(self, doc_ids: list, n_streams: int, seed: int):
        if n_streams < 1:
            raise ValueError("need n_streams >= 1")
        docs = [np.asarray(d, dtype=np.int64) for d in doc_ids if np.asarray(d).size]
        if not docs:
            raise ValueError("empty corpus")
        rng = np.random.default_rng(seed)
        if len(docs) >= n_streams:  # deal documents round-robin after a seeded shuffle
            order = rng.permutation(len(docs))
            groups = [[docs[i] for i in order[s::n_streams]] for s in range(n_streams)]
        else:  # one long text: N contiguous pieces
            total = np.concatenate(docs)
            if total.size < n_streams:
                raise ValueError(f"{total.size} tokens cannot fill {n_streams} streams")
            groups = [[part] for part in np.array_split(total, n_streams)]
        flat, cursors, base = [], [], 0
        for s, g in enumerate(groups):
            lengths = np.array([d.size for d in g], dtype=np.int64)
            starts = base + np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
            base += int(lengths.sum())
            flat.extend(g)
            cursors.append(_TapeCursor(lengths, starts, seed + 1000 + s))
        self.n_streams = n_streams
        self.corpus = np.concatenate(flat)
        self._cursors = cursors

    def next_positions(self, h_prime: int) -> tuple[np.ndarray, np.ndarray]:
        """(n_streams, h'+1) corpus positions (inputs then the look-ahead) and
        the new-document flags of this chunk."""
        n = self.n_streams
        pos = np.empty((n, h_prime + 1), dtype=np.int64)
        new_seq = np.zeros(n, dtype=bool)
        for s, cur in enumerate(self._cursors):
            pos[s], new_seq[s] = cur.read(h_prime)
        return pos, new_seq


class DeviceStreamSet:
    """StreamSource for train_loop with the corpus on the device."""

    def __init__(self, doc_ids: list, n_streams: int, seed: int):
        self._plan = TapePlanner(doc_ids, n_streams, seed)
        self.n_streams = n_streams
        self._corpus = torch.as_tensor(self._plan.corpus).to("cuda")
        self._lib = _lib.lib()

    def next_batch(self, h_prime: int) -> DeviceChunk:
        n = self.n_streams
        pos, new_seq = self._plan.next_positions(h_prime)
        dpos = torch.as_tensor(pos).to("cuda")
        inputs = torch.empty(h_prime * n, dtype=torch.int64, device="cuda")
        targets = torch.empty_like(inputs)
        P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(self._lib.rgb_tape_gather(P(self._corpus), P(dpos), P(inputs), P(targets), n, h_prime, st))
        return DeviceChunk(inputs=inputs, targets=targets, new_sequence=new_seq)
