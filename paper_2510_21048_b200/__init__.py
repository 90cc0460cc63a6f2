"""paper_2510_21048_b200 -- B200-native batched caching-allocator trace replay.

Thin ctypes binding over libxmem.so (include/xmem.h): argument marshalling
only. Every step of the hot path runs in the library's CUDA kernels; there is
no Python or CPU fallback -- on a GPU box, a missing or unloadable library is
a hard error. PyTorch is used for device memory and streams only.

    tr  = load_traces(bytes, tag, off)          # xm_load_traces (host, validated)
    dev = tr.to_device()                        # torch device tensors
    res = simulate_batch(dev, Config())         # xm_simulate_batch -> uint8[T, 64] on device
    pk  = peaks(res)                            # xm_peaks -> dict of numpy arrays
    pk  = simulate_host(tr, Config())           # end to end with host buffers (xm_simulate_host)

Widened rows, same conventions:
    dev = expand_templates(Templates(...), tpl, b, seed, thr)   # config 5 on device (K4)
    partner, mismatch, rec, wire = reconstruct(DeviceInstants.from_host(...))   # NEXT-3 (K5)
    cls, seq, rec, wire = orchestrate(DeviceProfiles.from_host(...))           # NEXT-2 (K6)
    m = metrics(runs)                                                          # NEXT-4
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Dict, Optional

import numpy as np

from . import _build

__all__ = ["Config", "Traces", "DeviceBatch", "load_traces", "simulate_batch", "peaks",
           "simulate_host", "simulate_raw", "Templates", "expand_templates", "lib", "XMemError", "RESULT_DTYPE", "FIELDS", "UNLIMITED"]

UNLIMITED = 0xFFFFFFFFFFFFFFFF
XM_FULL, XM_ALLOCATED_ONLY = 0, 1
STATUS = {0: "ok", 1: "oom", 2: "overflow"}
XM_O_OK, XM_O_FEW_ITERATIONS, XM_O_TS_RANGE = 0, 1, 2      # xm_orchestrated.status

# numpy view of xm_result (64 B, include/xmem.h)
RESULT_DTYPE = np.dtype([
    ("peak_allocated", "<u8"), ("peak_allocated_blk", "<u8"), ("peak_reserved", "<u8"),
    ("final_reserved", "<u8"), ("peak_allocated_idx", "<u4"), ("peak_allocated_blk_idx", "<u4"),
    ("peak_reserved_idx", "<u4"), ("n_seg_alloc", "<u4"), ("n_seg_release", "<u4"),
    ("max_live_segments", "<u4"), ("events_done", "<u4"), ("status", "<u2"),
    ("n_free_blocks_end", "<u2")])
assert RESULT_DTYPE.itemsize == 64
FIELDS = list(RESULT_DTYPE.names)


class XMemError(RuntimeError):
    pass


class _Cfg(ctypes.Structure):
    _fields_ = [("min_block", ctypes.c_uint64), ("small_size", ctypes.c_uint64),
                ("small_buffer", ctypes.c_uint64), ("large_buffer", ctypes.c_uint64),
                ("min_large_alloc", ctypes.c_uint64), ("round_large", ctypes.c_uint64),
                ("capacity", ctypes.c_uint64), ("large_split_strict", ctypes.c_uint32),
                ("mode", ctypes.c_uint32), ("smem_per_warp", ctypes.c_uint32),
                ("warps_per_cta", ctypes.c_uint32), ("roundup_power2_divisions", ctypes.c_uint32),
                ("reclaim_policy", ctypes.c_uint32), ("host_input", ctypes.c_uint32),
                ("_pad0", ctypes.c_uint32), ("max_split_size", ctypes.c_uint64),
                ("max_non_split_rounding", ctypes.c_uint64),
                ("garbage_collection_threshold", ctypes.c_double)]


class _Batch(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_void_p), ("tag", ctypes.c_void_p), ("off", ctypes.c_void_p),
                ("n_ids", ctypes.c_void_p), ("order", ctypes.c_void_p),
                ("capacity", ctypes.c_void_p), ("n_traces", ctypes.c_int64),
                ("n_events", ctypes.c_int64), ("max_ids", ctypes.c_uint32),
                ("max_events", ctypes.c_uint32), ("curve", ctypes.c_void_p),
                ("packed", ctypes.c_void_p)]


class _Summary(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in
                ("n_traces", "events_done", "n_oom", "n_overflow", "max_peak_reserved",
                 "max_peak_allocated", "sum_peak_reserved", "n_predicted_oom")]


class _Metrics(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("n_mre", ctypes.c_uint64), ("mre", ctypes.c_double),
                ("pef1", ctypes.c_double), ("pef2", ctypes.c_double), ("mcp", ctypes.c_double),
                ("sum_save", ctypes.c_int64), ("sum_c1", ctypes.c_uint64), ("sum_c2", ctypes.c_uint64)]


# xm_run (include/xmem.h): one evaluated run, 40 B
RUN_DTYPE = np.dtype([("m_peak_est", "<u8"), ("m_peak_meas1", "<u8"), ("m_peak_meas2", "<u8"),
                      ("m_max", "<u8"), ("oom_pred", "u1"), ("oom1", "u1"), ("oom2", "u1"),
                      ("_pad", "u1", (5,))])
assert RUN_DTYPE.itemsize == 40
ROUND2_NOT_RUN = 2


class _Instants(ctypes.Structure):
    _fields_ = [("addr", ctypes.c_void_p), ("bytes", ctypes.c_void_p), ("stream", ctypes.c_void_p),
                ("off", ctypes.c_void_p), ("n_traces", ctypes.c_int64), ("n_events", ctypes.c_int64),
                ("max_events", ctypes.c_uint32)]


# xm_lifecycle (include/xmem.h): per-trace reconstruction tallies, 64 B
LIFECYCLE_DTYPE = np.dtype([("n_blocks", "<u8"), ("n_orphan", "<u8"), ("n_mismatch", "<u8"),
                            ("n_persistent", "<u8"), ("n_kept", "<u8"), ("n_invalid", "<u8"),
                            ("max_open", "<u4"), ("n_ids", "<u4"), ("n_reopened", "<u8")])
assert LIFECYCLE_DTYPE.itemsize == 64


class _Profiles(ctypes.Structure):
    _fields_ = [("alloc_ts", ctypes.c_void_p), ("free_ts", ctypes.c_void_p), ("size", ctypes.c_void_p),
                ("stream", ctypes.c_void_p), ("boff", ctypes.c_void_p), ("win", ctypes.c_void_p),
                ("woff", ctypes.c_void_p), ("n_traces", ctypes.c_int64), ("n_blocks", ctypes.c_int64),
                ("max_blocks", ctypes.c_uint32)]


# xm_orchestrated (include/xmem.h), 56 B
ORCH_DTYPE = np.dtype([("ws", "<i8"), ("we", "<i8"), ("n_events", "<u8"), ("n_ids", "<u4"),
                       ("status", "<u4"), ("n_class", "<u4", (6,))])
assert ORCH_DTYPE.itemsize == 56


class _Tpl(ctypes.Structure):
    _fields_ = [("fixed", ctypes.c_void_p), ("per", ctypes.c_void_p), ("tag", ctypes.c_void_p),
                ("tpl_off", ctypes.c_void_p), ("n_tpl", ctypes.c_int64)]


@dataclass
class Config:
    """xm_config (include/xmem.h); defaults = torch CUDACachingAllocator constants."""
    min_block: int = 512
    small_size: int = 1 << 20
    small_buffer: int = 2 << 20
    large_buffer: int = 20 << 20
    min_large_alloc: int = 10 << 20
    round_large: int = 2 << 20
    capacity: int = UNLIMITED
    large_split_strict: int = 1
    mode: int = XM_FULL
    smem_per_warp: int = 0
    warps_per_cta: int = 0
    roundup_power2_divisions: int = 0     # NEXT-4 variant: torch knob (0/1 = off)
    reclaim_policy: int = 0               # 0 torch release-all; 1 SPEC.md:283 D3
    host_input: int = 0                   # xm_simulate_host: 0 auto, 1 direct, 2 stream, 3 copy
    _pad0: int = 0
    max_split_size: int = UNLIMITED       # torch max_split_size_mb:N -> N << 20 (Q26); off
    max_non_split_rounding: int = 20 << 20   # torch max_non_split_rounding_mb (Q26)
    garbage_collection_threshold: float = 0.0    # torch knob (Q27); 0 = off

    def c(self) -> _Cfg:
        return _Cfg(self.min_block, self.small_size, self.small_buffer, self.large_buffer,
                    self.min_large_alloc, self.round_large, self.capacity,
                    self.large_split_strict, self.mode, self.smem_per_warp, self.warps_per_cta,
                    self.roundup_power2_divisions, self.reclaim_policy, self.host_input, 0,
                    self.max_split_size, self.max_non_split_rounding,
                    self.garbage_collection_threshold)


_lib = None


def lib():
    """Load libxmem.so (building it in-tree if stale). Fails loudly."""
    global _lib
    if _lib is None:
        path = os.environ.get("XM_LIB") or _build.LIB    # XM_LIB: A/B tooling only
        if not os.path.exists(path) or os.environ.get("XM_REBUILD"):
            _build.build()
        L = ctypes.CDLL(path)
        P, I64, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64
        L.xm_config_default.argtypes = [P]
        L.xm_load_traces.argtypes = [P, P, P, I64, ctypes.POINTER(P), ctypes.POINTER(I64)]
        L.xm_traces_views.argtypes = [P] * 6 + [ctypes.POINTER(I64), ctypes.POINTER(I64),
                                                ctypes.POINTER(ctypes.c_uint32),
                                                ctypes.POINTER(ctypes.c_uint32)]
        L.xm_traces_packed.argtypes = [P, ctypes.POINTER(P)]
        L.xm_free_traces.argtypes = [P]
        L.xm_free_traces.restype = None
        L.xm_scratch_bytes.argtypes = [ctypes.POINTER(_Batch), ctypes.POINTER(_Cfg)]
        L.xm_scratch_bytes.restype = ctypes.c_size_t
        L.xm_simulate_batch.argtypes = [ctypes.POINTER(_Batch), ctypes.POINTER(_Cfg), P,
                                        ctypes.c_size_t, P, P]
        L.xm_peaks.argtypes = [P, I64, P, ctypes.POINTER(_Summary), U64, P]
        L.xm_host_ws_bytes.argtypes = [P, ctypes.POINTER(_Cfg)]
        L.xm_host_ws_bytes.restype = ctypes.c_size_t
        L.xm_simulate_host.argtypes = [P, P, ctypes.POINTER(_Cfg), P, ctypes.c_size_t, P, P]
        L.xm_raw_ws_bytes.argtypes = [P, ctypes.c_int64, ctypes.POINTER(_Cfg)]
        L.xm_raw_ws_bytes.restype = ctypes.c_size_t
        L.xm_simulate_raw.argtypes = [P, P, P, ctypes.c_int64, P, ctypes.POINTER(_Cfg), P,
                                      ctypes.c_size_t, P, ctypes.POINTER(ctypes.c_int64), P]
        L.xm_metrics_scratch_bytes.argtypes = [I64]
        L.xm_metrics_scratch_bytes.restype = ctypes.c_size_t
        L.xm_metrics_batch.argtypes = [P, I64, P, ctypes.c_size_t, ctypes.POINTER(_Metrics), P]
        L.xm_reconstruct_scratch_bytes.argtypes = [ctypes.POINTER(_Instants)]
        L.xm_reconstruct_scratch_bytes.restype = ctypes.c_size_t
        L.xm_reconstruct.argtypes = [ctypes.POINTER(_Instants), P, ctypes.c_size_t] + [P] * 4
        L.xm_reconstruct_wire.argtypes = [ctypes.POINTER(_Instants), P, ctypes.c_size_t] + [P] * 7
        L.xm_orchestrate_scratch_bytes.argtypes = [ctypes.POINTER(_Profiles)]
        L.xm_orchestrate_scratch_bytes.restype = ctypes.c_size_t
        L.xm_orchestrate.argtypes = [ctypes.POINTER(_Profiles), ctypes.c_uint32, P, ctypes.c_size_t,
                                     P, P, P, P]
        L.xm_orchestrate_wire.argtypes = [ctypes.POINTER(_Profiles), P, ctypes.c_size_t] + [P] * 7
        L.xm_blocks_from_instants.argtypes = [ctypes.POINTER(_Instants)] + [P] * 8
        L.xm_expand_templates.argtypes = [ctypes.POINTER(_Tpl), P, P, P, U64, P, I64, P, P, P, P]
        L.xm_last_error.restype = ctypes.c_char_p
        L.xm_last_launch_count.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().xm_last_error().decode(errors="replace")
        raise XMemError(f"{what} failed ({rc}): {msg}")


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Traces:
    """A validated, renumbered, packed host batch (xm_traces, page-locked),
    stored in processing (longest-first) order; results stay in caller order."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        L = lib()
        ptrs = [ctypes.c_void_p() for _ in range(5)]
        nt, ne = ctypes.c_int64(), ctypes.c_int64()
        mi, me = ctypes.c_uint32(), ctypes.c_uint32()
        _check(L.xm_traces_views(handle, *[ctypes.byref(p) for p in ptrs], ctypes.byref(nt),
                                 ctypes.byref(ne), ctypes.byref(mi), ctypes.byref(me)),
               "xm_traces_views")
        self.n_traces, self.n_events = nt.value, ne.value
        self.max_ids, self.max_events = mi.value, me.value

        def view(p, dt, n):
            if n == 0:
                return np.zeros(0, dt)
            buf = (ctypes.c_char * (np.dtype(dt).itemsize * n)).from_address(p.value)
            return np.frombuffer(buf, dt, n)
        self.bytes = view(ptrs[0], np.int64, self.n_events)
        self.tag = view(ptrs[1], np.uint32, self.n_events)
        self.off = view(ptrs[2], np.int64, self.n_traces + 1)
        self.n_ids = view(ptrs[3], np.uint32, self.n_traces)
        self.order = view(ptrs[4], np.uint32, self.n_traces)
        # the batch is STORED longest-first: stored trace i is the caller's
        # trace order[i], its events are [off[i], off[i+1]); pos[t] = i
        self.pos = np.empty(self.n_traces, np.int64)
        self.pos[self.order.astype(np.int64)] = np.arange(self.n_traces)
        pk = ctypes.c_void_p()
        _check(L.xm_traces_packed(handle, ctypes.byref(pk)), "xm_traces_packed")
        self.packed = view(pk, np.uint64, self.n_events) if pk.value else None

    def span(self, t: int):
        """Event range [a, b) of the caller's trace t in the stored arrays
        (and in a memory-curve output)."""
        i = int(self.pos[t])
        return int(self.off[i]), int(self.off[i + 1])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.xm_free_traces(h)
            self._h = None

    def to_device(self, device=None, capacity: Optional[np.ndarray] = None,
                  non_blocking: bool = False, packed: bool = False) -> "DeviceBatch":
        """Device copy; packed=True uploads the compact 8-byte events
        (xm_batch.packed) instead of bytes + tag."""
        import torch
        device = torch.device(device or "cuda")

        def t(a):
            return torch.from_numpy(a).to(device, non_blocking=non_blocking)
        cap = None
        if capacity is not None:
            cap = torch.from_numpy(np.ascontiguousarray(capacity, np.uint64).view(np.int64)).to(
                device, non_blocking=non_blocking)
        if packed:
            if self.packed is None:
                raise XMemError("no packed form: an id space exceeds 2^18")
            db = DeviceBatch(None, None, t(self.off), t(self.n_ids.view(np.int32)),
                             t(self.order.view(np.int32)), cap, self.n_traces, self.n_events,
                             self.max_ids, self.max_events)
            db.packed = t(self.packed.view(np.int64))
            return db
        return DeviceBatch(t(self.bytes), t(self.tag.view(np.int32)), t(self.off),
                           t(self.n_ids.view(np.int32)), t(self.order.view(np.int32)), cap,
                           self.n_traces, self.n_events, self.max_ids, self.max_events)


@dataclass
class DeviceBatch:
    bytes: "object"
    tag: "object"
    off: "object"
    n_ids: "object"
    order: "object"
    capacity: "object"
    n_traces: int
    n_events: int
    max_ids: int
    max_events: int
    _scratch: Dict = field(default_factory=dict)
    packed: "object" = None              # optional compact events (xm_batch.packed)

    def c(self, curve=None) -> _Batch:
        def p(x):
            return ctypes.c_void_p(x.data_ptr()) if x is not None and x.numel() else None
        return _Batch(p(self.bytes), p(self.tag), p(self.off), p(self.n_ids), p(self.order),
                      p(self.capacity), self.n_traces, self.n_events, self.max_ids,
                      self.max_events, p(curve), p(self.packed))


def load_traces(bytes_: np.ndarray, tag: np.ndarray, off: np.ndarray) -> Traces:
    """xm_load_traces: validate + renumber + pack host traces."""
    b = np.ascontiguousarray(bytes_, np.int64)
    g = np.ascontiguousarray(tag, np.uint32)
    o = np.ascontiguousarray(off, np.int64)
    h = ctypes.c_void_p()
    bad = ctypes.c_int64(-1)
    rc = lib().xm_load_traces(_np_ptr(b), _np_ptr(g), _np_ptr(o), len(o) - 1, ctypes.byref(h),
                              ctypes.byref(bad))
    if rc != 0:
        msg = lib().xm_last_error().decode(errors="replace")
        err = XMemError(f"xm_load_traces failed ({rc}) at trace {bad.value}: {msg}")
        err.code, err.trace = rc, bad.value
        raise err
    return Traces(h)


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def scratch_bytes(dev: DeviceBatch, cfg: Config = Config()) -> int:
    b, c = dev.c(), cfg.c()
    return int(lib().xm_scratch_bytes(ctypes.byref(b), ctypes.byref(c)))


def simulate_batch(dev: DeviceBatch, cfg: Config = Config(), stream=None, out=None, curve=None):
    """xm_simulate_batch on the current (or given) torch stream.
    Returns a uint8 device tensor [n_traces, 64] holding xm_result records.
    curve: optional int64 device tensor [n_events, 3] receiving the memory-usage
    curve (allocated, allocated blocks, reserved bytes after each event), rows
    in stored event order (Traces.span(t) gives trace t's rows)."""
    import torch
    if curve is not None:
        assert curve.dtype == torch.int64 and curve.shape == (dev.n_events, 3) and curve.is_contiguous()
    b, c = dev.c(curve), cfg.c()
    need = int(lib().xm_scratch_bytes(ctypes.byref(b), ctypes.byref(c)))
    key = (cfg.mode, cfg.smem_per_warp, cfg.warps_per_cta)
    scr = dev._scratch.get(key)
    if scr is None or scr.numel() < need:
        scr = torch.empty(max(need, 256), dtype=torch.uint8, device=dev.off.device)
        dev._scratch[key] = scr
    if out is None:
        out = torch.empty((dev.n_traces, 64), dtype=torch.uint8, device=dev.off.device)
    rc = lib().xm_simulate_batch(ctypes.byref(b), ctypes.byref(c), ctypes.c_void_p(scr.data_ptr()),
                                 scr.numel(), ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream))
    _check(rc, "xm_simulate_batch")
    return out


def last_launch_count() -> int:
    return int(lib().xm_last_launch_count())


def peaks(res, capacity_for_eq1: int = UNLIMITED, stream=None):
    """xm_peaks: device results -> (structured numpy array, summary dict)."""
    n = res.shape[0]
    h = np.zeros(n, RESULT_DTYPE)
    s = _Summary()
    rc = lib().xm_peaks(ctypes.c_void_p(res.data_ptr()), n, _np_ptr(h), ctypes.byref(s),
                        ctypes.c_uint64(capacity_for_eq1), _stream_ptr(stream))
    _check(rc, "xm_peaks")
    return h, {k: int(getattr(s, k)) for k, _ in _Summary._fields_}


def simulate_host(tr: Traces, cfg: Config = Config(), capacity: Optional[np.ndarray] = None,
                  stream=None, workspace=None):
    """xm_simulate_host: host buffers in, host results out (H2D + replay + D2H)."""
    import torch
    c = cfg.c()
    need = int(lib().xm_host_ws_bytes(tr._h, ctypes.byref(c)))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device="cuda")
    h = np.zeros(tr.n_traces, RESULT_DTYPE)
    cap = None
    if capacity is not None:
        cap = np.ascontiguousarray(capacity, np.uint64)
    rc = lib().xm_simulate_host(tr._h, _np_ptr(cap) if cap is not None else None, ctypes.byref(c),
                                ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                _np_ptr(h), _stream_ptr(stream))
    _check(rc, "xm_simulate_host")
    return h, workspace


def simulate_raw(bytes_: np.ndarray, tag: np.ndarray, off: np.ndarray, cfg: Config = Config(),
                 capacity: Optional[np.ndarray] = None, stream=None, workspace=None):
    """xm_simulate_raw: the caller's raw host arrays (xm_load_traces' contract)
    validated, renumbered and replayed on the device; results (numpy
    RESULT_DTYPE, caller order) and the workspace for reuse. Page-locked
    arrays (e.g. numpy views of pinned torch tensors) are read in place.
    Raises XMemError (with .bad_trace) on an invalid trace."""
    import torch
    by = np.ascontiguousarray(bytes_, np.int64)
    tg = np.ascontiguousarray(tag, np.uint32)
    of = np.ascontiguousarray(off, np.int64)
    T = len(of) - 1
    c = cfg.c()
    need = int(lib().xm_raw_ws_bytes(_np_ptr(of), T, ctypes.byref(c)))
    if need == 0:
        _check(-1, "xm_raw_ws_bytes")
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device="cuda")
    h = np.zeros(T, RESULT_DTYPE)
    cap = None if capacity is None else np.ascontiguousarray(capacity, np.uint64)
    bad = ctypes.c_int64(-1)
    rc = lib().xm_simulate_raw(_np_ptr(by), _np_ptr(tg), _np_ptr(of), T,
                               _np_ptr(cap) if cap is not None else None, ctypes.byref(c),
                               ctypes.c_void_p(workspace.data_ptr()), workspace.numel(), _np_ptr(h),
                               ctypes.byref(bad), _stream_ptr(stream))
    if rc != 0:
        msg = lib().xm_last_error().decode(errors="replace")
        err = XMemError(f"xm_simulate_raw failed ({rc}): {msg}")
        err.bad_trace = bad.value
        raise err
    return h, workspace


def as_dict(h: np.ndarray) -> Dict[str, np.ndarray]:
    return {k: h[k].astype(np.uint64) for k in FIELDS}


# ---- config 5: on-device template expansion (xm_expand_templates, K4) --------
class Templates:
    """A device-resident template pool (xm_templates): per-event signed fixed
    and per-sample bytes, tags with dense ids, offsets, id space per template."""

    def __init__(self, fixed, per, tag, tpl_off, n_ids, device=None):
        import torch
        device = torch.device(device or "cuda")
        self.fixed = torch.from_numpy(np.ascontiguousarray(fixed, np.int64)).to(device)
        self.per = torch.from_numpy(np.ascontiguousarray(per, np.int64)).to(device)
        self.tag = torch.from_numpy(np.ascontiguousarray(tag, np.uint32).view(np.int32)).to(device)
        self.tpl_off = torch.from_numpy(np.ascontiguousarray(tpl_off, np.int64)).to(device)
        self.h_off = np.ascontiguousarray(tpl_off, np.int64)
        self.n_ids = np.ascontiguousarray(n_ids, np.uint32)
        self.n_tpl = len(self.h_off) - 1
        self.device = device

    def c(self) -> _Tpl:
        return _Tpl(ctypes.c_void_p(self.fixed.data_ptr()), ctypes.c_void_p(self.per.data_ptr()),
                    ctypes.c_void_p(self.tag.data_ptr()), ctypes.c_void_p(self.tpl_off.data_ptr()),
                    self.n_tpl)


def expand_templates(tp: Templates, tpl: np.ndarray, b: np.ndarray, seed: np.ndarray,
                     swap_threshold: int, capacity: Optional[np.ndarray] = None, stream=None,
                     check: bool = True, reuse: Optional[DeviceBatch] = None) -> DeviceBatch:
    """Build a DeviceBatch of len(tpl) traces (caller order = the given order)
    entirely on the device with xm_expand_templates. Traces are stored
    longest-first (ties in caller order), like xm_load_traces stores them.
    reuse: a DeviceBatch of the same descriptors whose event arrays are
    rewritten in place (no allocation)."""
    import torch
    tpl = np.ascontiguousarray(tpl, np.uint32)
    n = len(tpl)
    lens = np.diff(tp.h_off)[tpl]
    order = np.argsort(-lens, kind="stable").astype(np.uint32)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(lens[order])
    nids = tp.n_ids[tpl][order]
    dev = tp.device

    def t(a, dt, view=None):
        a = np.ascontiguousarray(a, dt)
        return torch.from_numpy(a.view(view) if view else a).to(dev)
    d_tpl = t(tpl[order], np.uint32, np.int32)
    d_b = t(np.asarray(b)[order], np.uint32, np.int32)
    d_seed = t(np.asarray(seed)[order], np.uint64, np.int64)
    d_off = t(off, np.int64)
    n_ev = int(off[-1])
    if reuse is not None:
        assert reuse.n_events == n_ev and reuse.n_traces == n
        d_bytes, d_tag = reuse.bytes, reuse.tag
    else:
        d_bytes = torch.empty(n_ev, dtype=torch.int64, device=dev)
        d_tag = torch.empty(n_ev, dtype=torch.int32, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    args = (d_tpl, d_b, d_seed, d_off, flag, int(swap_threshold))
    _launch_expand(tp, args, n, d_bytes, d_tag, stream)
    if check and int(flag.item()) != 0:
        raise XMemError("xm_expand_templates: template lengths disagree with offsets")
    cap = None
    if capacity is not None:
        cap = t(np.asarray(capacity, np.uint64), np.uint64, np.int64)
    db = DeviceBatch(d_bytes, d_tag, d_off, t(nids, np.uint32, np.int32),
                     t(order, np.uint32, np.int32), cap, n, n_ev,
                     int(nids.max()) if n else 0, int(lens.max()) if n else 0)
    db._scratch["k4"] = args
    return db


def _launch_expand(tp: Templates, args, n, d_bytes, d_tag, stream):
    d_tpl, d_b, d_seed, d_off, flag, thr = args
    c = tp.c()

    def p(x):
        return ctypes.c_void_p(x.data_ptr()) if x.numel() else None
    rc = lib().xm_expand_templates(ctypes.byref(c), p(d_tpl), p(d_b), p(d_seed),
                                   ctypes.c_uint64(thr), p(d_off), n, p(d_bytes), p(d_tag),
                                   ctypes.c_void_p(flag.data_ptr()), _stream_ptr(stream))
    _check(rc, "xm_expand_templates")


def expand_again(tp: Templates, db: DeviceBatch, stream=None):
    """Re-run K4 into db's event arrays with its resident descriptors (one
    launch, nothing else: used to time the kernel)."""
    _launch_expand(tp, db._scratch["k4"], db.n_traces, db.bytes, db.tag, stream)


# ---- NEXT-4: batched evaluation metrics (xm_metrics_batch) ----------------------
def metrics(runs, stream=None) -> Dict[str, float]:
    """MRE / PEF / MCP of N runs. runs: numpy RUN_DTYPE array
    (copied to the device) or a uint8 device tensor [N, 40]."""
    import torch
    if isinstance(runs, np.ndarray):
        assert runs.dtype == RUN_DTYPE
        d = torch.from_numpy(np.ascontiguousarray(runs).view(np.uint8).reshape(-1, 40)).cuda()
    else:
        d = runs
    n = d.shape[0]
    need = int(lib().xm_metrics_scratch_bytes(n))
    scr = torch.empty(max(need, 256), dtype=torch.uint8, device=d.device)
    m = _Metrics()
    rc = lib().xm_metrics_batch(ctypes.c_void_p(d.data_ptr()) if n else None, n,
                                ctypes.c_void_p(scr.data_ptr()), scr.numel(), ctypes.byref(m),
                                _stream_ptr(stream))
    _check(rc, "xm_metrics_batch")
    return {k: getattr(m, k) for k, _ in _Metrics._fields_}


# ---- NEXT-3: lifecycle reconstruction (xm_reconstruct) ---------------------------
@dataclass
class DeviceInstants:
    addr: "object"        # uint64 as int64 tensor [E]
    bytes: "object"       # int64 [E]
    stream: "object"      # uint8 [E] or None
    off: "object"         # int64 [T+1]
    n_traces: int
    n_events: int
    max_events: int

    @staticmethod
    def from_host(addr, bytes_, stream, off, device=None) -> "DeviceInstants":
        import torch
        device = torch.device(device or "cuda")
        off = np.ascontiguousarray(off, np.int64)
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).to(device)
        lens = np.diff(off)
        return DeviceInstants(t(np.asarray(addr, np.uint64).view(np.int64), np.int64),
                              t(bytes_, np.int64),
                              t(stream, np.uint8) if stream is not None else None, t(off, np.int64),
                              len(off) - 1, int(off[-1]), int(lens.max()) if len(lens) else 0)

    def c(self) -> _Instants:
        def p(x):
            return ctypes.c_void_p(x.data_ptr()) if x is not None and x.numel() else None
        return _Instants(p(self.addr), p(self.bytes), p(self.stream), p(self.off), self.n_traces,
                         self.n_events, self.max_events)


def reconstruct(ins: DeviceInstants, wire: bool = True, stream=None, scratch=None):
    """xm_reconstruct: partner / mismatch (device int32 / uint8 tensors), the
    per-trace tallies (numpy LIFECYCLE_DTYPE) and, with wire=True, the replay
    batch the reconstruction defines (DeviceBatch, stored in trace order)."""
    import torch
    dev = ins.off.device
    c = ins.c()
    need = int(lib().xm_reconstruct_scratch_bytes(ctypes.byref(c)))
    if scratch is None or scratch.numel() < need:
        scratch = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
    E, T = ins.n_events, ins.n_traces
    partner = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    mism = torch.empty(max(E, 1), dtype=torch.uint8, device=dev)
    rec = torch.empty((max(T, 1), LIFECYCLE_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    wb = wt = wo = wn = None
    if wire:
        wb = torch.empty(max(E, 1), dtype=torch.int64, device=dev)
        wt = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
        wo = torch.empty(T + 1, dtype=torch.int64, device=dev)
        wn = torch.empty(max(T, 1), dtype=torch.int32, device=dev)

    def p(x):
        return ctypes.c_void_p(x.data_ptr()) if x is not None else None
    rc = lib().xm_reconstruct(ctypes.byref(c), ctypes.c_void_p(scratch.data_ptr()), scratch.numel(),
                              p(partner), p(mism), p(rec), _stream_ptr(stream))
    _check(rc, "xm_reconstruct")
    r = rec[:T].cpu().numpy().reshape(-1).view(LIFECYCLE_DTYPE) if T else np.zeros(0, LIFECYCLE_DTYPE)
    batch = None
    if wire:
        # stored longest first (ties in trace order), like xm_load_traces stores
        order_h = np.argsort(-r["n_kept"].astype(np.int64), kind="stable").astype(np.uint32)
        order = torch.from_numpy(order_h.view(np.int32)).to(dev)
        rc = lib().xm_reconstruct_wire(ctypes.byref(c), ctypes.c_void_p(scratch.data_ptr()),
                                       scratch.numel(), p(rec), p(order), p(wb), p(wt), p(wo),
                                       p(wn), _stream_ptr(stream))
        _check(rc, "xm_reconstruct_wire")
        n_wire = int(r["n_kept"].sum()) if T else 0
        if T and int(r["n_ids"].max()) > (1 << 27):
            raise XMemError("xm_reconstruct: a trace keeps more than 2^27 blocks open; its wire "
                            "trace exceeds the replay's id space (include/xmem.h XM_ID_BITS)")
        batch = DeviceBatch(wb[:max(n_wire, 0)], wt[:max(n_wire, 0)], wo, wn[:T], order, None, T,
                            n_wire, int(r["n_ids"].max()) if T else 0,
                            int(r["n_kept"].max()) if T else 0)
    return partner[:E], mism[:E], r, batch


# ---- NEXT-2: memory orchestrator (xm_orchestrate) --------------------------------
@dataclass
class DeviceProfiles:
    alloc_ts: "object"
    free_ts: "object"
    size: "object"
    stream: "object"
    boff: "object"
    win: "object"
    woff: "object"
    n_traces: int
    n_blocks: int
    max_blocks: int

    @staticmethod
    def from_host(p, device=None) -> "DeviceProfiles":
        """p: workloads.cpu_profile.Profiles (or any object with its fields)."""
        import torch
        device = torch.device(device or "cuda")
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).to(device)
        boff = np.ascontiguousarray(p.boff, np.int64)
        lens = np.diff(boff)
        return DeviceProfiles(t(p.alloc_ts, np.int64), t(p.free_ts, np.int64), t(p.size, np.int64),
                              t(p.stream, np.uint8) if p.stream is not None else None, t(boff, np.int64),
                              t(np.asarray(p.win, np.int64).reshape(-1), np.int64), t(p.woff, np.int64),
                              len(boff) - 1, int(boff[-1]), int(lens.max()) if len(lens) else 0)

    def c(self) -> _Profiles:
        def p(x):
            return ctypes.c_void_p(x.data_ptr()) if x is not None and x.numel() else None
        return _Profiles(p(self.alloc_ts), p(self.free_ts), p(self.size), p(self.stream), p(self.boff),
                         p(self.win), p(self.woff), self.n_traces, self.n_blocks, self.max_blocks)


def orchestrate(prof: DeviceProfiles, analysis_iter: int = 1, wire: bool = True, stream=None,
                scratch=None):
    """xm_orchestrate (+ xm_orchestrate_wire): classes (device uint8 [n_blocks]),
    sorted sequences (device uint64 keys, trace t at 2*boff[t]), per-trace
    records (numpy ORCH_DTYPE) and, with wire=True, the replay batch of the
    re-timed sequences stored longest first (DeviceBatch)."""
    import torch
    dev = prof.boff.device
    c = prof.c()
    need = int(lib().xm_orchestrate_scratch_bytes(ctypes.byref(c)))
    if scratch is None or scratch.numel() < need:
        scratch = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
    B, T = prof.n_blocks, prof.n_traces
    cls = torch.empty(max(B, 1), dtype=torch.uint8, device=dev)
    seq = torch.empty(max(2 * B, 1), dtype=torch.int64, device=dev)
    rec = torch.empty((max(T, 1), 56), dtype=torch.uint8, device=dev)

    def p(x):
        return ctypes.c_void_p(x.data_ptr()) if x is not None else None
    rc = lib().xm_orchestrate(ctypes.byref(c), analysis_iter, ctypes.c_void_p(scratch.data_ptr()),
                              scratch.numel(), p(cls), p(seq), p(rec), _stream_ptr(stream))
    _check(rc, "xm_orchestrate")
    r = rec[:T].cpu().numpy().reshape(-1).view(ORCH_DTYPE) if T else np.zeros(0, ORCH_DTYPE)
    batch = None
    if wire:
        n_ev = r["n_events"].astype(np.int64)
        order_h = np.argsort(-n_ev, kind="stable").astype(np.uint32)
        order = torch.from_numpy(order_h.view(np.int32)).to(dev)
        n_wire = int(n_ev.sum())
        wb = torch.empty(max(n_wire, 1), dtype=torch.int64, device=dev)
        wt = torch.empty(max(n_wire, 1), dtype=torch.int32, device=dev)
        wo = torch.empty(T + 1, dtype=torch.int64, device=dev)
        wn = torch.empty(max(T, 1), dtype=torch.int32, device=dev)
        rc = lib().xm_orchestrate_wire(ctypes.byref(c), ctypes.c_void_p(scratch.data_ptr()),
                                       scratch.numel(), p(rec), p(order), p(wb), p(wt), p(wo), p(wn),
                                       _stream_ptr(stream))
        _check(rc, "xm_orchestrate_wire")
        batch = DeviceBatch(wb[:n_wire], wt[:n_wire], wo, wn[:T], order, None, T, n_wire,
                            int(r["n_ids"].max()) if T else 0, int(n_ev.max()) if T else 0)
    return cls[:B], seq, r, batch


# ---- the GPU pipeline: instants -> blocks -> orchestrated sequence -> peaks --------
def blocks_from_instants(ins: DeviceInstants, ts, partner, rec, stream=None) -> "DeviceProfiles":
    """xm_blocks_from_instants: the reconstruction's blocks (allocation order)
    as an orchestrator input without windows (set .win / .woff before use)."""
    import torch
    dev = ins.off.device
    nb = rec["n_blocks"].astype(np.int64) if len(rec) else np.zeros(0, np.int64)
    boff = np.zeros(ins.n_traces + 1, np.int64)
    boff[1:] = np.cumsum(nb)
    B = int(boff[-1])
    d_boff = torch.from_numpy(boff).to(dev)
    a = torch.empty(max(B, 1), dtype=torch.int64, device=dev)
    f = torch.empty(max(B, 1), dtype=torch.int64, device=dev)
    z = torch.empty(max(B, 1), dtype=torch.int64, device=dev)
    st = torch.empty(max(B, 1), dtype=torch.uint8, device=dev)
    c = ins.c()

    def p(x):
        return ctypes.c_void_p(x.data_ptr()) if x is not None and x.numel() else None
    rc = lib().xm_blocks_from_instants(ctypes.byref(c), p(ts), p(partner), p(d_boff), p(a), p(f),
                                       p(z), p(st), _stream_ptr(stream))
    _check(rc, "xm_blocks_from_instants")
    return DeviceProfiles(a[:B], f[:B], z[:B], st[:B], d_boff, None, None, ins.n_traces, B,
                          int(nb.max()) if len(nb) else 0)


def estimate(ins: DeviceInstants, ts, win: np.ndarray, woff: np.ndarray, analysis_iter: int = 1,
             cfg: Config = Config(), capacity: Optional[np.ndarray] = None, stream=None,
             curve: bool = False):
    """xMem's pipeline on the GPU (Fig. 3 after profiling; SPEC.md:296
    estimate, without the operator attribution): profiler instants -> lifecycle
    reconstruction (K5) -> blocks -> memory orchestrator (K6) -> replay (K2) ->
    per-trace results. win [iters, 6, 2] / woff [T+1]: the annotation windows.
    curve=True adds the memory-usage curve of the re-timed sequences (P:205
    "an optional detailed memory usage curve"; rows in the wire batch's stored
    order: details["wire"].off / .order locate trace t).
    Returns (results numpy RESULT_DTYPE in trace order, summary, details)."""
    import torch
    dev = ins.off.device
    partner, mism, rec, _ = reconstruct(ins, wire=False, stream=stream)
    prof = blocks_from_instants(ins, ts, partner, rec, stream=stream)
    prof.win = torch.from_numpy(np.ascontiguousarray(win, np.int64).reshape(-1)).to(dev)
    prof.woff = torch.from_numpy(np.ascontiguousarray(woff, np.int64)).to(dev)
    cls, seq, orec, wb = orchestrate(prof, analysis_iter, stream=stream)
    bad = np.flatnonzero(orec["status"] != XM_O_OK) if len(orec) else np.zeros(0, np.int64)
    if len(bad):
        # SPEC.md:300-304 (insufficient iterations is an error) and the
        # orchestrator's range checks: such a trace has no valid re-timed
        # sequence, so it must not be replayed as if it were empty
        t = int(bad[0])
        raise XMemError(f"estimate: {len(bad)} trace(s) not orchestrated; first trace {t} "
                        f"status {int(orec['status'][t])} "
                        f"({'fewer than analysis_iter + 1 iterations' if orec['status'][t] == XM_O_FEW_ITERATIONS else 'timestamp or size out of range'})")
    if capacity is not None:
        wb.capacity = torch.from_numpy(np.ascontiguousarray(capacity, np.uint64).view(np.int64)).to(dev)
    cv = None
    if curve:
        cv = torch.zeros((wb.n_events, 3), dtype=torch.int64, device=dev)
    res = simulate_batch(wb, cfg, stream, curve=cv)
    h, summ = peaks(res, stream=stream)
    return h, summ, {"lifecycle": rec, "orchestrated": orec, "classes": cls, "profiles": prof,
                     "wire": wb, "curve": cv}
