"""The oracle on all host cores -- test infrastructure (tests/ and bench.py's
cpu_baseline / --impl reference legs only).

Workers are FORKED processes that inherit their inputs through module globals
set before the pool starts: nothing but chunk numbers is pickled on the way in
(the round-1 pool pickled every chunk's event arrays, which made 16 processes
only ~3x one core). Each worker times only the oracle's simulate call; a run
reports both the wall time of the whole pool pass and the busiest worker's
simulate time ("timing only simulate").

Two jobs:
  * run(batch)            -- oracle results of every trace (+ timings);
  * parity_mc5(idx, h)    -- config 5 at full size: each worker rebuilds its
                             chunk of Monte-Carlo traces on the host
                             (workloads.mc5.batch_fast), replays it with the
                             oracle and compares every field with the GPU's
                             results h (caller order), returning only counts.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

import oracle
from workloads.trace import Batch

# fields compared bit-exactly (tests/gpu_util.py COMPARE; n_free_blocks_end saturates)
COMPARE = ["peak_allocated", "peak_allocated_idx", "peak_allocated_blk", "peak_allocated_blk_idx",
           "peak_reserved", "peak_reserved_idx", "final_reserved", "n_seg_alloc",
           "n_seg_release", "max_live_segments", "events_done", "status", "n_free_blocks_end"]

_G: dict = {}


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _bounds(off: np.ndarray, chunks: int):
    """Contiguous trace ranges with ~equal event counts."""
    T = len(off) - 1
    E = int(off[-1])
    cut = [0] + [int(np.searchsorted(off[1:], E * k / chunks)) for k in range(1, chunks)] + [T]
    cut = sorted(set(min(max(c, 0), T) for c in cut))
    return [(a, z) for a, z in zip(cut[:-1], cut[1:]) if z > a]


def _sim_chunk(i):
    a, z = _G["bounds"][i]
    b = _G["batch"]
    ea, ez = int(b.off[a]), int(b.off[z])
    sub = Batch(b.bytes[ea:ez], b.tag[ea:ez], b.off[a:z + 1] - ea, b.capacity[a:z])
    t0 = time.perf_counter()
    o = oracle.simulate_batch(sub, _G["cfg"])
    dt = time.perf_counter() - t0
    return i, os.getpid(), dt, o


class Pool:
    """A fork pool over one batch. Reusable: every pass re-runs the oracle on
    the inherited batch (the reference arm's steps)."""

    def __init__(self, batch, cfg: oracle.Config = oracle.Config(), workers: int = 0,
                 chunks_per_worker: int = 4):
        self.workers = workers or host_cores()
        _G.clear()
        _G["batch"] = batch
        _G["cfg"] = cfg
        _G["bounds"] = _bounds(batch.off, max(1, self.workers * chunks_per_worker))
        self.n = len(_G["bounds"])
        self.pool = mp.get_context("fork").Pool(self.workers)

    def run(self):
        """One pass. Returns (results dict, wall s, busiest worker's simulate s,
        summed simulate s)."""
        t0 = time.perf_counter()
        parts = [None] * self.n
        per_worker = {}
        total = 0.0
        for i, pid, dt, o in self.pool.imap_unordered(_sim_chunk, range(self.n)):
            parts[i] = o
            per_worker[pid] = per_worker.get(pid, 0.0) + dt
            total += dt
        wall = time.perf_counter() - t0
        res = {k: np.concatenate([p[k] for p in parts]) for k in oracle.FIELDS}
        return res, wall, max(per_worker.values()), total

    def close(self):
        self.pool.close()
        self.pool.join()
        _G.clear()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def run(batch, cfg: oracle.Config = oracle.Config(), workers: int = 0):
    """Oracle results of every trace of `batch` on all host cores."""
    if batch.n_traces < 2:
        return oracle.simulate_batch(batch, cfg)
    with Pool(batch, cfg, workers) as p:
        return p.run()[0]


# ---- config 5 at full size ------------------------------------------------------
def _mc5_chunk(i):
    from workloads import mc5
    idx = _G["idx"][_G["bounds"][i][0]:_G["bounds"][i][1]]
    t0 = time.perf_counter()
    hb = mc5.batch_fast(idx)
    t1 = time.perf_counter()
    o = oracle.simulate_batch(hb)
    t2 = time.perf_counter()
    h = _G["h"]
    pos = _G["pos"][_G["bounds"][i][0]:_G["bounds"][i][1]]
    bad = {}
    first = -1
    for f in COMPARE:
        exp = o[f].astype(np.uint64)
        if f == "n_free_blocks_end":
            exp = np.minimum(exp, 65535)
        got = h[f][pos].astype(np.uint64)
        m = np.flatnonzero(got != exp)
        if len(m):
            bad[f] = int(len(m))
            first = int(idx[m[0]]) if first < 0 else min(first, int(idx[m[0]]))
    return (i, os.getpid(), len(idx), int(o["events_done"].sum()), int((o["status"] == 1).sum()),
            t1 - t0, t2 - t1, bad, first)


def parity_mc5(idx: np.ndarray, h: np.ndarray, pos: np.ndarray = None, workers: int = 0,
               chunk_traces: int = 2000):
    """Compare the GPU results h (numpy RESULT_DTYPE) of config-5 traces idx
    (h[pos[k]] is trace idx[k]; pos defaults to idx) with the oracle, every
    trace, every field. Returns a summary dict."""
    idx = np.asarray(idx, np.int64)
    workers = workers or host_cores()
    _G.clear()
    _G["idx"] = idx
    _G["h"] = h
    _G["pos"] = idx if pos is None else np.asarray(pos, np.int64)
    _G["bounds"] = [(a, min(a + chunk_traces, len(idx))) for a in range(0, len(idx), chunk_traces)]
    n = len(_G["bounds"])
    t0 = time.perf_counter()
    traces = events = ooms = 0
    gen = sim = 0.0
    per_worker = {}
    bad: dict = {}
    first = -1
    with mp.get_context("fork").Pool(workers) as pool:
        for i, pid, nt, ev, no, dg, ds, b, f in pool.imap_unordered(_mc5_chunk, range(n)):
            traces += nt
            events += ev
            ooms += no
            gen += dg
            sim += ds
            per_worker[pid] = per_worker.get(pid, 0.0) + ds
            for k, v in b.items():
                bad[k] = bad.get(k, 0) + v
            if f >= 0:
                first = f if first < 0 else min(first, f)
    wall = time.perf_counter() - t0
    _G.clear()
    return {"traces": traces, "fields": len(COMPARE), "mismatched_values": int(sum(bad.values())),
            "mismatched_by_field": bad, "first_mismatch_trace": first, "oracle_events": events,
            "oracle_oom_traces": ooms, "workers": workers, "wall_s": wall,
            "oracle_simulate_s_max_worker": max(per_worker.values()) if per_worker else 0.0,
            "host_generation_s_total": gen, "oracle_simulate_s_total": sim}
