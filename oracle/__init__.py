"""ORACLE -- test infrastructure only.

Plain CPU reference of xMem's Simulator (§3.4) written in C
(``oracle/xmo.c``) and loaded here with ctypes. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. It shares no code with
``paper_2510_21048_b200`` (the product) and never imports it.

Contents: the Simulator (``xmo.c``; allocator variants of NEXT-4 included),
lifecycle reconstruction (``lifecycle.c``, NEXT-3; ``reconstruct`` /
``wire_from_partner`` below), and in plain Python the Memory Orchestrator
(``orchestrator.py``, NEXT-2) and the evaluation metrics (``metrics.py``,
NEXT-4).

Parity status: all functions pinned (tests/test_oracle_pins.py,
tests/test_oracle_bruteforce.py, tests/test_oracle_variants.py,
tests/test_oracle_lifecycle.py, tests/test_oracle_orchestrator.py,
tests/test_oracle_metrics.py, and the mutation checks in
tests/test_oracle_mutants.py); see DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "xmo.c")
_SRCS = [_SRC, os.path.join(_HERE, "lifecycle.c")]
_LIB = os.path.join(_HERE, "libxmo.so")

FIELDS = ["peak_allocated", "peak_allocated_idx", "peak_allocated_blk", "peak_allocated_blk_idx",
          "peak_reserved", "peak_reserved_idx", "final_reserved", "n_seg_alloc", "n_seg_release",
          "max_live_segments", "events_done", "status", "n_free_blocks_end",
          "final_allocated", "final_allocated_blk"]
NF = len(FIELDS)
UNLIMITED = 0xFFFFFFFFFFFFFFFF
MiB = 1 << 20

ERRORS = {-1: "zero-byte request", -2: "alloc of a live id", -3: "free of a non-live id",
          -4: "free size differs from alloc", -5: "out of host memory", -6: "invariant violated"}


class OracleError(RuntimeError):
    def __init__(self, code, trace=-1):
        super().__init__(f"oracle error {code} ({ERRORS.get(code, '?')}) in trace {trace}")
        self.code = code
        self.trace = trace


class _Cfg(ctypes.Structure):
    _fields_ = [("min_block", ctypes.c_uint64), ("small_size", ctypes.c_uint64),
                ("small_buffer", ctypes.c_uint64), ("large_buffer", ctypes.c_uint64),
                ("min_large_alloc", ctypes.c_uint64), ("round_large", ctypes.c_uint64),
                ("capacity", ctypes.c_uint64), ("large_split_strict", ctypes.c_int32),
                ("roundup_power2_divisions", ctypes.c_int32), ("reclaim_policy", ctypes.c_int32),
                ("_pad", ctypes.c_int32), ("max_split_size", ctypes.c_uint64),
                ("max_non_split_rounding", ctypes.c_uint64), ("gc_threshold", ctypes.c_double)]


@dataclass
class Config:
    """SPEC.md:210 SimConfig; defaults = the torch constants the paper defers to."""
    min_block: int = 512
    small_size: int = 1 * MiB
    small_buffer: int = 2 * MiB
    large_buffer: int = 20 * MiB
    min_large_alloc: int = 10 * MiB
    round_large: int = 2 * MiB
    capacity: int = UNLIMITED
    large_split_strict: int = 1
    roundup_power2_divisions: int = 0    # NEXT-4 variant (torch knob); 0/1 = off
    reclaim_policy: int = 0              # 0 torch release-all (Q3); 1 SPEC.md:283 D3
    max_split_size: int = UNLIMITED      # torch max_split_size_mb:N -> N MiB (Q26); off
    max_non_split_rounding: int = 20 * MiB   # torch max_non_split_rounding_mb (Q26)
    gc_threshold: float = 0.0            # torch garbage_collection_threshold (Q27); off

    def c(self) -> _Cfg:
        return _Cfg(self.min_block, self.small_size, self.small_buffer, self.large_buffer,
                    self.min_large_alloc, self.round_large, self.capacity,
                    self.large_split_strict, self.roundup_power2_divisions,
                    self.reclaim_policy, 0, self.max_split_size, self.max_non_split_rounding,
                    self.gc_threshold)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or \
            os.path.getmtime(_LIB) < max(os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC",
                               "-o", tmp, *_SRCS])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.xmo_simulate.argtypes = [P, P, ctypes.c_int64, ctypes.POINTER(_Cfg), ctypes.c_uint64,
                                   P, P, ctypes.c_int]
        L.xmo_simulate_batch.argtypes = [P, P, P, ctypes.c_int64, ctypes.POINTER(_Cfg), P, P,
                                         ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]
        for f in ("xmo_round_size", "xmo_segment_size"):
            getattr(L, f).argtypes = [ctypes.c_uint64, ctypes.POINTER(_Cfg)]
            getattr(L, f).restype = ctypes.c_uint64
        L.xmo_is_small.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Cfg)]
        L.xmo_should_split.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(_Cfg)]
        L.xmo_reconstruct.argtypes = [P, P, ctypes.c_int64, P, P, P]
        assert L.xmo_nfields() == NF
        _lib = L
    return _lib


def round_size(req: int, cfg: Config = Config()) -> int:
    c = cfg.c()
    return int(lib().xmo_round_size(req, ctypes.byref(c)))


def segment_size(s: int, cfg: Config = Config()) -> int:
    c = cfg.c()
    return int(lib().xmo_segment_size(s, ctypes.byref(c)))


def is_small(s: int, cfg: Config = Config()) -> bool:
    c = cfg.c()
    return bool(lib().xmo_is_small(s, ctypes.byref(c)))


def should_split(small: bool, rem: int, cfg: Config = Config()) -> bool:
    c = cfg.c()
    return bool(lib().xmo_should_split(int(small), rem, ctypes.byref(c)))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def simulate_trace(bytes_: np.ndarray, tag: np.ndarray, capacity: int = UNLIMITED,
                   cfg: Config = Config(), curve: bool = False, check: bool = False):
    """One trace. Returns (dict of fields, curve[n,3] or None)."""
    b = np.ascontiguousarray(bytes_, np.int64)
    g = np.ascontiguousarray(tag, np.uint32)
    out = np.zeros(NF, np.uint64)
    cv = np.zeros((len(b), 3), np.uint64) if curve else None
    c = cfg.c()
    rc = lib().xmo_simulate(_ptr(b), _ptr(g), len(b), ctypes.byref(c), int(capacity), _ptr(out),
                            _ptr(cv) if cv is not None else None, int(check))
    if rc:
        raise OracleError(rc, 0)
    return {k: int(v) for k, v in zip(FIELDS, out)}, cv


def simulate_batch(batch, cfg: Config = Config(), check: bool = False) -> Dict[str, np.ndarray]:
    """All traces of a workloads.Batch, single-threaded. Returns field -> uint64[T]."""
    b = np.ascontiguousarray(batch.bytes, np.int64)
    g = np.ascontiguousarray(batch.tag, np.uint32)
    off = np.ascontiguousarray(batch.off, np.int64)
    cap = np.ascontiguousarray(batch.capacity, np.uint64)
    T = len(off) - 1
    out = np.zeros((T, NF), np.uint64)
    bad = ctypes.c_int64(-1)
    c = cfg.c()
    rc = lib().xmo_simulate_batch(_ptr(b), _ptr(g), _ptr(off), T, ctypes.byref(c), _ptr(cap),
                                  _ptr(out), int(check), ctypes.byref(bad))
    if rc:
        raise OracleError(rc, bad.value)
    return {k: out[:, i].copy() for i, k in enumerate(FIELDS)}


def _worker(args):
    b, g, off, cap, cfgd = args
    from workloads.trace import Batch
    return simulate_batch(Batch(b, g, off, cap), Config(**cfgd))


def simulate_batch_parallel(batch, cfg: Config = Config(), workers: Optional[int] = None,
                            chunks: int = 0) -> Dict[str, np.ndarray]:
    """Same result as simulate_batch, traces split over host processes."""
    import multiprocessing as mp
    from dataclasses import asdict
    workers = workers or os.cpu_count() or 1
    T = batch.n_traces
    if workers <= 1 or T < 2:
        return simulate_batch(batch, cfg)
    chunks = chunks or min(T, workers * 4)
    # contiguous chunks with ~equal event counts
    cum = batch.off[1:]
    bounds = [0]
    for k in range(1, chunks):
        bounds.append(int(np.searchsorted(cum, batch.n_events * k / chunks)))
    bounds.append(T)
    bounds = sorted(set(bounds))
    jobs = []
    for a, z in zip(bounds[:-1], bounds[1:]):
        if z <= a:
            continue
        ea, ez = int(batch.off[a]), int(batch.off[z])
        jobs.append((batch.bytes[ea:ez], batch.tag[ea:ez], batch.off[a:z + 1] - ea,
                     batch.capacity[a:z], asdict(cfg)))
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        parts = pool.map(_worker, jobs)
    return {k: np.concatenate([p[k] for p in parts]) for k in FIELDS}


# ---- lifecycle reconstruction (oracle/lifecycle.c) -------------
LIFECYCLE_TALLIES = ["n_blocks", "n_orphan", "n_mismatch", "n_persistent", "n_kept", "max_open"]


def reconstruct(addr: np.ndarray, bytes_: np.ndarray):
    """One trace of instants -> (partner int64[n], mismatch uint8[n], tallies dict)."""
    a = np.ascontiguousarray(addr, np.uint64)
    b = np.ascontiguousarray(bytes_, np.int64)
    n = len(b)
    partner = np.zeros(n, np.int64)
    mism = np.zeros(n, np.uint8)
    t = np.zeros(6, np.uint64)
    rc = lib().xmo_reconstruct(_ptr(a), _ptr(b), n, _ptr(partner), _ptr(mism), _ptr(t))
    if rc:
        raise OracleError(rc, 0)
    return partner, mism, {k: int(v) for k, v in zip(LIFECYCLE_TALLIES, t)}


def wire_from_partner(bytes_: np.ndarray, stream: np.ndarray, partner: np.ndarray):
    """The replay input a reconstruction defines (the definition, written out):
    kept events = allocations + matched frees, in order; an allocation keeps
    its bytes and stream, a matched free becomes -(its block's size) on its
    block's stream (the wire contract, include/xmem.h xm_batch); block ids =
    allocation ordinals. Returns (bytes', tag', kept index)."""
    b = np.asarray(bytes_, np.int64)
    st = np.asarray(stream, np.uint32)
    is_alloc = b > 0
    kept = np.flatnonzero(is_alloc | (partner >= 0))
    ordinal = np.cumsum(is_alloc) - 1
    out_b = np.where(is_alloc[kept], b[kept], -b[np.maximum(partner[kept], 0)])
    blk = np.where(is_alloc[kept], kept, partner[kept])
    out_t = (ordinal[blk].astype(np.uint32) | (st[blk] << np.uint32(28))).astype(np.uint32)
    return out_b.astype(np.int64), out_t, kept
