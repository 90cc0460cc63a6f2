"""Memory-instant streams (the profiler's cpu_instant_event records: address,
signed bytes, time order) for the lifecycle-reconstruction row
(SURVEY.md §8(f) NEXT-3). Input generation only.

A trace of alloc/free events with block ids is given CPU-allocator-like
addresses: a freed address goes back to a per-size LIFO free list and is
reused by the next allocation of that size, else a bump pointer (64 B
aligned) -- so addresses are reused the way P:217 ("correctly handling
address reuse") expects. Seeded noise emulates imperfect traces (SPEC.md:110
"orphan-free tally", "mismatch tally"):
  p_orphan    an extra free of an address that was never allocated
  p_mismatch  a free whose |bytes| differs from its allocation
  p_lost      a free that was not recorded (its block stays open, but the
              address is still recycled: later allocations stack on it)
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np

from .rng import generator, trace_seed
from .trace import Batch


@dataclass
class Instants:
    addr: np.ndarray       # uint64[E]
    bytes: np.ndarray      # int64[E]   + alloc, - free
    stream: np.ndarray     # uint8[E]
    off: np.ndarray        # int64[T+1]
    names: List[str] = field(default_factory=list)

    @property
    def n_traces(self) -> int:
        return int(len(self.off) - 1)

    @property
    def n_events(self) -> int:
        return int(self.off[-1])

    def trace(self, t: int):
        a, b = int(self.off[t]), int(self.off[t + 1])
        return self.addr[a:b], self.bytes[a:b], self.stream[a:b]


def from_trace(by, tg, seed: int, p_orphan=0.0, p_mismatch=0.0, p_lost=0.0):
    g = generator(seed)
    n = len(by)
    u = g.random((n, 3))
    base = 0x7F0000000000 + (int(g.integers(0, 1 << 20)) << 12)
    bump = base
    free_lists = {}
    where = {}
    A, B, S = [], [], []
    for i in range(n):
        b = int(by[i])
        bid = int(tg[i]) & 0x0FFFFFFF
        st = int(tg[i]) >> 28
        if u[i, 0] < p_orphan:                          # a stray free
            A.append(bump + (1 << 40))
            B.append(-int(g.integers(1, 1 << 20)))
            S.append(st)
        if b > 0:
            fl = free_lists.get(b)
            if fl:
                a = fl.pop()
            else:
                a = bump
                bump += (b + 63) // 64 * 64
            where[bid] = a
            A.append(a)
            B.append(b)
            S.append(st)
        else:
            a = where.pop(bid)
            free_lists.setdefault(-b, []).append(a)
            if u[i, 1] < p_lost:
                continue                                   # free not recorded
            nb = b
            if u[i, 2] < p_mismatch:
                nb = b - int(g.integers(1, 512))           # recorded size differs
            A.append(a)
            B.append(nb)
            S.append(st)
    return (np.asarray(A, np.uint64), np.asarray(B, np.int64), np.asarray(S, np.uint8))


def from_batch(batch: Batch, salt: int = 11, **noise) -> Instants:
    parts = [from_trace(*batch.trace(t), seed=trace_seed(t, salt), **noise)
             for t in range(batch.n_traces)]
    off = np.zeros(len(parts) + 1, np.int64)
    off[1:] = np.cumsum([len(p[0]) for p in parts])
    cat = (lambda k, dt: np.concatenate([p[k] for p in parts]) if parts else np.zeros(0, dt))
    return Instants(cat(0, np.uint64), cat(1, np.int64), cat(2, np.uint8), off,
                    list(batch.names) if batch.names else [])
