"""Trace containers in the SoA wire format (see package docstring)."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

UNLIMITED = np.uint64(0xFFFFFFFFFFFFFFFF)
ID_BITS = 28
ID_MASK = (1 << ID_BITS) - 1
MAX_STREAMS = 16


@dataclass
class Batch:
    bytes: np.ndarray      # int64[E]
    tag: np.ndarray        # uint32[E]
    off: np.ndarray        # int64[T+1]
    capacity: np.ndarray   # uint64[T]
    names: List[str] = field(default_factory=list)

    @property
    def n_traces(self) -> int:
        return int(self.off.shape[0] - 1)

    @property
    def n_events(self) -> int:
        return int(self.off[-1])

    def trace(self, t: int):
        a, b = int(self.off[t]), int(self.off[t + 1])
        return self.bytes[a:b], self.tag[a:b]

    def lengths(self) -> np.ndarray:
        return np.diff(self.off)

    def subset(self, idx: Sequence[int]) -> "Batch":
        idx = list(idx)
        parts_b, parts_t, lens = [], [], []
        for t in idx:
            b, g = self.trace(t)
            parts_b.append(b)
            parts_t.append(g)
            lens.append(len(b))
        off = np.zeros(len(idx) + 1, np.int64)
        off[1:] = np.cumsum(lens)
        names = [self.names[t] for t in idx] if self.names else []
        return Batch(np.concatenate(parts_b) if parts_b else np.zeros(0, np.int64),
                     np.concatenate(parts_t) if parts_t else np.zeros(0, np.uint32),
                     off, self.capacity[idx].copy(), names)


def concat(batches: Sequence[Batch]) -> Batch:
    bs = [b for b in batches]
    off = [np.zeros(1, np.int64)]
    base = 0
    for b in bs:
        off.append(b.off[1:] + base)
        base += b.n_events
    return Batch(np.concatenate([b.bytes for b in bs]) if bs else np.zeros(0, np.int64),
                 np.concatenate([b.tag for b in bs]) if bs else np.zeros(0, np.uint32),
                 np.concatenate(off),
                 np.concatenate([b.capacity for b in bs]) if bs else np.zeros(0, np.uint64),
                 sum((b.names for b in bs), []))


class TraceBuilder:
    """Accumulates one or more traces event by event (small/hand-built traces)."""

    def __init__(self):
        self._bytes: List[int] = []
        self._tag: List[int] = []
        self._off: List[int] = [0]
        self._cap: List[int] = []
        self._names: List[str] = []
        self._live = {}

    def alloc(self, bid: int, nbytes: int, stream: int = 0):
        assert 0 <= bid <= ID_MASK and 0 <= stream < MAX_STREAMS and nbytes > 0
        self._live[bid] = nbytes
        self._bytes.append(int(nbytes))
        self._tag.append(bid | (stream << ID_BITS))
        return self

    def free(self, bid: int, stream: Optional[int] = None):
        nbytes = self._live.pop(bid)
        self._bytes.append(-int(nbytes))
        self._tag.append(bid | ((stream or 0) << ID_BITS))
        return self

    def end_trace(self, capacity: Optional[int] = None, name: str = ""):
        self._off.append(len(self._bytes))
        self._cap.append(int(UNLIMITED) if capacity is None else int(capacity))
        self._names.append(name)
        self._live = {}
        return self

    def build(self) -> Batch:
        return Batch(np.asarray(self._bytes, np.int64), np.asarray(self._tag, np.uint32),
                     np.asarray(self._off, np.int64), np.asarray(self._cap, np.uint64),
                     list(self._names))


def from_arrays(bytes_: np.ndarray, tag: np.ndarray, capacity=None, name: str = "") -> Batch:
    off = np.array([0, len(bytes_)], np.int64)
    cap = np.array([int(UNLIMITED) if capacity is None else int(capacity)], np.uint64)
    return Batch(np.asarray(bytes_, np.int64), np.asarray(tag, np.uint32), off, cap, [name])
