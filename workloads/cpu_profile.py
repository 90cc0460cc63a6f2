"""CPU-profile-shaped block traces for the orchestrator row (SURVEY.md §8(f)
NEXT-2): what the Analyzer hands the Memory Orchestrator (PAPER.md:226
"size, initial CPU-based allocation and deallocation timestamps"; SPEC.md
MemoryBlock) plus the training-loop annotation windows it uses (PAPER.md:212
"profiler.step() ... optimizer.zero_grad()"). Input generation only.

From a template with phase markers (models.template_phases): event j gets
CPU time ts_j = 10 (j + 1) + jitter (0-4 us); a marker before position p is
at 10 p + 7. The capture covers the template's iterations (3) and ends
at the last iteration's end: later frees (teardown) are not seen, so
parameters and optimizer state come out persistent. CPU-vs-GPU divergence the
orchestrator exists to undo: a batch tensor is freed on the CPU
only when the next batch is loaded (Python rebinding), i.e. inside the next
iteration's data window (or never, after the last one).

Per trace: blocks in allocation order (alloc_ts, free_ts or -1, size, stream,
and the generator's ground-truth kind -- for reporting only), and per
iteration six windows [start, end]: iteration, data, forward, backward,
zero_grad (-1, -1 if absent), optimizer.step.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import models as M
from .rng import generator, trace_seed

WINDOWS = ["iter", "data", "fw", "bw", "zg", "opt"]
KINDS = ["param", "data", "act", "grad", "state", "temp"]


@dataclass
class Profiles:
    alloc_ts: np.ndarray     # int64[B]
    free_ts: np.ndarray      # int64[B]  -1 = no deallocation observed
    size: np.ndarray         # int64[B]
    stream: np.ndarray       # uint8[B]
    kind: np.ndarray         # uint8[B]  ground truth (KINDS index), reporting only
    boff: np.ndarray         # int64[T+1] blocks of trace t
    win: np.ndarray          # int64[I, 6, 2] windows per iteration
    woff: np.ndarray         # int64[T+1] iterations of trace t
    names: List[str] = field(default_factory=list)

    @property
    def n_traces(self) -> int:
        return len(self.boff) - 1

    def trace(self, t):
        a, b = int(self.boff[t]), int(self.boff[t + 1])
        c, d = int(self.woff[t]), int(self.woff[t + 1])
        return (self.alloc_ts[a:b], self.free_ts[a:b], self.size[a:b], self.stream[a:b],
                self.win[c:d])


def profile(name, opt, zg, b, seed, streams=False, img=32, seq=512):
    (sign, fixed, per, bid, stream), marks, kinds = M.template_phases(
        name, opt, zg, streams=streams, img=img, seq=seq)
    g = generator(seed)
    n = len(sign)
    ts = 10 * (np.arange(n, dtype=np.int64) + 1) + g.integers(0, 5, n)
    mts = {}
    its = []
    cur = None
    for (m, p) in marks:
        t = 10 * p + 7
        if m == "iter_start":
            cur = {"iter": [t, -1]}
            its.append(cur)
        elif m.endswith("_start"):
            cur[m[:-6]] = [t, -1]
        else:
            key = m[:-4]
            cur[key][1] = t
    end = its[-1]["iter"][1]
    win = np.full((len(its), 6, 2), -1, np.int64)
    for k, it in enumerate(its):
        for w, key in enumerate(WINDOWS):
            if key in it:
                win[k, w] = it[key]
    # pair events into blocks (allocation order)
    alloc_pos = {}
    blocks = []
    for j in range(n):
        if sign[j] > 0:
            alloc_pos[int(bid[j])] = len(blocks)
            blocks.append([int(ts[j]), -1, int(fixed[j] + per[j] * b), int(stream[j]),
                           KINDS.index(kinds[len(blocks)])])
        else:
            k = alloc_pos.pop(int(bid[j]))
            if ts[j] < end:
                blocks[k][1] = int(ts[j])
    blocks = [x for x in blocks if x[0] < end]            # allocated inside the capture
    # batch data freed when the next batch is loaded (CPU-side divergence)
    data_starts = win[:, 1, 0]
    for x in blocks:
        if KINDS[x[4]] == "data":
            nxt = data_starts[data_starts > x[0]]
            later = nxt[nxt > win[np.searchsorted(win[:, 0, 0], x[0], side="right") - 1, 0, 1]]
            x[1] = int(later[0]) + 1 + int(g.integers(0, 3)) if len(later) else -1
    arr = np.asarray(blocks, np.int64).reshape(-1, 5)
    return arr, win


def batch(cells, salt: int = 12) -> Profiles:
    """cells: [(model, optimizer, zero_grad, batch size, streams)]"""
    parts, wins = [], []
    for t, (name, opt, zg, b, streams) in enumerate(cells):
        arr, win = profile(name, opt, zg, b, trace_seed(t, salt), streams=streams)
        parts.append(arr)
        wins.append(win)
    boff = np.zeros(len(parts) + 1, np.int64)
    boff[1:] = np.cumsum([len(p) for p in parts])
    woff = np.zeros(len(wins) + 1, np.int64)
    woff[1:] = np.cumsum([len(w) for w in wins])
    cat = np.concatenate(parts) if parts else np.zeros((0, 5), np.int64)
    return Profiles(cat[:, 0].copy(), cat[:, 1].copy(), cat[:, 2].copy(), cat[:, 3].astype(np.uint8),
                    cat[:, 4].astype(np.uint8), boff,
                    np.concatenate(wins) if wins else np.zeros((0, 6, 2), np.int64), woff,
                    ["/".join(map(str, c)) for c in cells])


def suite_cells(n: int, salt: int = 13):
    """n cells drawn like the paper's Monte Carlo configurations."""
    from . import suites
    out = []
    for i in range(n):
        name, opt, b, zg, cap, _ = suites.mc_draw(i, salt)
        out.append((name, opt, zg, b, False))
    return out


def to_instants(p: Profiles, salt: int = 17):
    """The profiler's memory instants behind a Profiles batch (PAPER.md:215
    cpu_instant_event: time, address, signed bytes): per trace, every block's
    allocation and (if observed) deallocation, in time order (ties in block
    order, allocation before deallocation of later blocks as generated), with
    CPU-allocator-like addresses (a freed address is reused LIFO by the next
    allocation of the same size, else a 64 B-aligned bump pointer).
    Returns (ts, addr, bytes, stream, off) numpy arrays."""
    T = p.n_traces
    TS, AD, BY, ST, off = [], [], [], [], [0]
    for t in range(T):
        a, f, s, st, _ = p.trace(t)
        ev = [(int(a[i]), 0, i, 1) for i in range(len(a))]
        ev += [(int(f[i]), 1, i, -1) for i in range(len(a)) if f[i] >= 0]
        ev.sort()
        g = generator(trace_seed(t, salt))
        bump = 0x7E0000000000 + (int(g.integers(0, 1 << 20)) << 12)
        free_lists, where = {}, {}
        for (ts, _, i, sign) in ev:
            sz = int(s[i])
            if sign > 0:
                fl = free_lists.get(sz)
                if fl:
                    ad = fl.pop()
                else:
                    ad = bump
                    bump += (sz + 63) // 64 * 64
                where[i] = ad
            else:
                ad = where.pop(i)
                free_lists.setdefault(sz, []).append(ad)
            TS.append(ts)
            AD.append(ad)
            BY.append(sign * sz)
            ST.append(int(st[i]))
        off.append(len(TS))
    return (np.asarray(TS, np.int64), np.asarray(AD, np.uint64), np.asarray(BY, np.int64),
            np.asarray(ST, np.uint8), np.asarray(off, np.int64))
