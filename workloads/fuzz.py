"""Random alloc/free sequences (SPEC.md:508 acceptance #1) and adversarial sets.

SPEC #1: "1,000 seeded random sequences (<=1,000 events each, sizes 1 B-64 MiB,
mixed alloc/free)". Recipe: sizes log-uniform over
[1 B, 64 MiB], P(alloc)=0.55, a free picks a uniformly random live block,
streams {0,1} in half the sequences, every sequence closed (all blocks freed at
the end, in random order). Block ids are arbitrary (not dense) and are reused
after their free with probability 1/4, to exercise the loader's renumbering.
"""
from __future__ import annotations

import math
from typing import Optional

import numpy as np

from .rng import generator, trace_seed
from .trace import Batch, ID_BITS, UNLIMITED, concat

MiB = 1 << 20


def random_trace(seed: int, max_events: int = 1000, max_bytes: int = 64 * MiB,
                 min_bytes: int = 1, p_alloc: float = 0.55, n_streams: int = 1,
                 closed: bool = True, capacity: Optional[int] = None,
                 name: str = "") -> Batch:
    rng = generator(seed)
    bytes_, tag = [], []
    live = {}          # id -> (bytes, stream)
    live_ids = []
    freed_ids = []
    next_id = int(rng.integers(0, 1 << 20))
    lo, hi = math.log(min_bytes), math.log(max_bytes)
    while len(bytes_) + (len(live) if closed else 0) < max_events:
        if not live or rng.random() < p_alloc:
            if freed_ids and rng.random() < 0.25:
                bid = freed_ids.pop(int(rng.integers(0, len(freed_ids))))
            else:
                bid = next_id
                next_id += int(rng.integers(1, 5))
            nb = int(math.exp(rng.uniform(lo, hi)))
            nb = max(min_bytes, min(max_bytes, nb))
            st = int(rng.integers(0, n_streams))
            live[bid] = (nb, st)
            live_ids.append(bid)
            bytes_.append(nb)
            tag.append(bid | (st << ID_BITS))
        else:
            k = int(rng.integers(0, len(live_ids)))
            bid = live_ids[k]
            live_ids[k] = live_ids[-1]
            live_ids.pop()
            nb, st = live.pop(bid)
            freed_ids.append(bid)
            bytes_.append(-nb)
            tag.append(bid | (st << ID_BITS))
    if closed:
        order = list(live_ids)
        rng.shuffle(order)
        for bid in order:
            nb, st = live.pop(bid)
            bytes_.append(-nb)
            tag.append(bid | (st << ID_BITS))
    cap = int(UNLIMITED) if capacity is None else int(capacity)
    return Batch(np.asarray(bytes_, np.int64), np.asarray(tag, np.uint32),
                 np.array([0, len(bytes_)], np.int64), np.array([cap], np.uint64), [name])


def spec1_corpus(n: int = 1000, max_events: int = 1000, salt: int = 1) -> Batch:
    """SPEC #1 corpus: n sequences; streams {0,1} in the odd-indexed half."""
    parts = []
    for i in range(n):
        s = trace_seed(i, salt)
        parts.append(random_trace(s, max_events=max_events,
                                  n_streams=2 if (i & 1) else 1,
                                  name=f"fuzz{salt}-{i}"))
    return concat(parts)


def small_size_corpus(n: int = 200, max_events: int = 400, salt: int = 2) -> Batch:
    """Sizes 1 B-4 MiB: exercises the small pool, splits and coalescing densely."""
    parts = [random_trace(trace_seed(i, salt), max_events=max_events, max_bytes=4 * MiB,
                          n_streams=1 + (i % 3), name=f"small{salt}-{i}") for i in range(n)]
    return concat(parts)


def capacity_corpus(n: int = 200, max_events: int = 600, salt: int = 3) -> Batch:
    """Finite capacity near the working set: exercises reclamation and OOM."""
    parts = []
    for i in range(n):
        cap = int(generator(trace_seed(i, salt + 100)).integers(8, 200)) * 2 * MiB
        parts.append(random_trace(trace_seed(i, salt), max_events=max_events,
                                  n_streams=1 + (i & 1), capacity=cap, name=f"cap{salt}-{i}"))
    return concat(parts)


def fragmentation_stress(n_allocs: int = 4096, size: int = 512, name="frag") -> Batch:
    """4096 x 512 B allocs, then free every other one -> 2048 free holes."""
    bytes_, tag = [], []
    for i in range(n_allocs):
        bytes_.append(size)
        tag.append(i)
    for i in range(0, n_allocs, 2):
        bytes_.append(-size)
        tag.append(i)
    # re-allocate into the holes with a mix of sizes, then close
    nid = n_allocs
    for i in range(n_allocs // 4):
        bytes_.append(size * (1 + (i % 3)))
        tag.append(nid + i)
    for i in range(n_allocs // 4):
        bytes_.append(-size * (1 + (i % 3)))
        tag.append(nid + i)
    for i in range(1, n_allocs, 2):
        bytes_.append(-size)
        tag.append(i)
    return Batch(np.asarray(bytes_, np.int64), np.asarray(tag, np.uint32),
                 np.array([0, len(bytes_)], np.int64), np.array([UNLIMITED], np.uint64), [name])
