"""The C-ABI library builds, loads, exports every declared symbol, and its
host-side logic (validation, renumbering, LPT order) is correct. No GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2510_21048_b200 as xm
from workloads import fuzz, hand
from workloads.trace import TraceBuilder

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "xmem.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(xm_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("xm_load_traces", "xm_simulate_batch", "xm_peaks", "xm_last_error",
                 "xm_scratch_bytes", "xm_traces_views", "xm_free_traces", "xm_simulate_host"):
        assert must in names


def test_library_exports_every_declared_symbol():
    L = xm.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
        assert ctypes.cast(getattr(L, name), ctypes.c_void_p).value


def test_result_struct_is_64_bytes():
    assert xm.RESULT_DTYPE.itemsize == 64


def test_config_default_matches_binding():
    c = xm._Cfg()
    xm.lib().xm_config_default(ctypes.byref(c))
    d = xm.Config()
    for f, _ in xm._Cfg._fields_:
        assert getattr(c, f) == getattr(d, f), f


def _max_live(by):
    return int(np.cumsum(np.sign(by)).max()) if len(by) else 0


def test_loader_renumbers_densely():
    c = fuzz.spec1_corpus(50, 500, salt=31)
    tr = xm.load_traces(c.bytes, c.tag, c.off)
    assert tr.n_traces == 50 and tr.n_events == c.n_events
    for t in range(c.n_traces):
        a, b = c.off[t], c.off[t + 1]
        sa, sb = tr.span(t)                                     # stored copy of trace t
        assert sb - sa == b - a
        by = c.bytes[a:b]
        assert (tr.bytes[sa:sb] == by).all()
        dense = tr.tag[sa:sb] & ((1 << 28) - 1)
        raw = c.tag[a:b] & ((1 << 28) - 1)
        # allocs keep their stream; a free carries its block's alloc stream
        st_in, st_out, alloc_stream = c.tag[a:b] >> 28, tr.tag[sa:sb] >> 28, {}
        for k in range(len(by)):
            if by[k] > 0:
                assert st_out[k] == st_in[k]
                alloc_stream[raw[k]] = st_in[k]
            else:
                assert st_out[k] == alloc_stream.pop(raw[k])
        i = int(tr.pos[t])
        assert tr.n_ids[i] == _max_live(by)
        assert dense.max() < tr.n_ids[i]
        # the renaming is a bijection between live raw ids and live dense ids
        live = {}
        for k in range(len(by)):
            if by[k] > 0:
                assert dense[k] not in live.values()
                live[raw[k]] = dense[k]
            else:
                assert live.pop(raw[k]) == dense[k]
    assert tr.max_ids == tr.n_ids.max()
    assert tr.max_events == np.diff(c.off).max()


def test_loader_lpt_order():
    """Stored order = processing order: longest first, ties in caller order;
    the stored arrays are the caller's traces permuted by order."""
    c = fuzz.spec1_corpus(40, 700, salt=32)
    tr = xm.load_traces(c.bytes, c.tag, c.off)
    L = np.diff(c.off)
    assert sorted(tr.order.tolist()) == list(range(40))
    assert (np.diff(L[tr.order]) <= 0).all()
    assert (np.diff(tr.off) == L[tr.order]).all() and tr.off[0] == 0
    for i in range(39):                                         # stable
        if L[tr.order[i]] == L[tr.order[i + 1]]:
            assert tr.order[i] < tr.order[i + 1]
    perm = np.concatenate([np.arange(c.off[t], c.off[t + 1]) for t in tr.order])
    assert (tr.bytes == c.bytes[perm]).all()


def test_loader_reports_first_bad_caller_trace():
    """With several invalid traces the smallest CALLER index is reported, even
    though traces are validated in (longest-first) storage order."""
    by = np.array([512, -512,            # 0 ok
                   512, -1024,           # 1 bad (short): free size mismatch
                   512, 512, 512, 512, 512], np.int64)   # 2 bad (long): alloc of a live id
    tg = np.array([1, 1, 1, 1, 1, 1, 1, 1, 1], np.uint32)

    class bt:
        bytes, tag, off = by, tg, np.array([0, 2, 4, 9], np.int64)
    with pytest.raises(xm.XMemError) as e:
        xm.load_traces(bt.bytes, bt.tag, bt.off)
    assert e.value.trace == 1


@pytest.mark.parametrize("events,code", [
    ([(0, 1)], -1),                    # zero-byte request
    ([(512, 1), (512, 1)], -1),        # alloc of a live id
    ([(-512, 1)], -1),                 # free of a non-live id
    ([(512, 1), (-1024, 1)], -1),      # free size mismatch
    ([(1 << 40, 1)], -4),              # request >= 2^40 (XM_ERANGE)
])
def test_loader_rejects(events, code):
    good = TraceBuilder().alloc(0, 100).free(0).end_trace().build()
    by = np.concatenate([good.bytes, np.array([e[0] for e in events], np.int64)])
    tg = np.concatenate([good.tag, np.array([e[1] for e in events], np.uint32)])
    off = np.array([0, 2, len(by)], np.int64)
    with pytest.raises(xm.XMemError) as e:
        xm.load_traces(by, tg, off)
    assert e.value.code == code and e.value.trace == 1


def test_loader_accepts_id_reuse_and_empty_traces():
    b = TraceBuilder()
    b.alloc(7, 100).free(7).alloc(7, 200).free(7).end_trace()
    b.end_trace()                                   # empty trace
    b.alloc(1 << 27, 5, stream=3).free(1 << 27, stream=3).end_trace()
    bt = b.build()
    tr = xm.load_traces(bt.bytes, bt.tag, bt.off)
    assert tr.n_ids[tr.pos].tolist() == [1, 0, 1]
    a, b = tr.span(2)
    assert (tr.tag[a:b] >> 28 == 3).all()


def test_loader_bad_offsets():
    with pytest.raises(xm.XMemError):
        xm.load_traces(np.array([5, -5], np.int64), np.zeros(2, np.uint32),
                       np.array([0, 2, 1], np.int64))


def test_simulate_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = hand.h1(512, 3)
    tr = xm.load_traces(c.bytes, c.tag, c.off)
    b = xm._Batch(None, None, None, None, None, None, tr.n_traces, tr.n_events, tr.max_ids,
                  tr.max_events)
    cfg = xm.Config().c()
    rc = xm.lib().xm_simulate_batch(ctypes.byref(b), ctypes.byref(cfg), None, 0, None, None)
    assert rc != 0


def test_scratch_sizing_is_host_only():
    c = fuzz.spec1_corpus(10, 300, salt=33)
    tr = xm.load_traces(c.bytes, c.tag, c.off)
    b = xm._Batch(None, None, None, None, None, None, tr.n_traces, tr.n_events, tr.max_ids,
                  tr.max_events)
    cfg = xm.Config().c()
    n = xm.lib().xm_scratch_bytes(ctypes.byref(b), ctypes.byref(cfg))
    assert n >= 256


def test_packed_events_encode_bytes_and_tags():
    """xm_load_traces also builds the compact 8-byte events (xm_batch.packed):
    they decode to exactly the stored bytes and tags."""
    c = fuzz.spec1_corpus(30, 400, salt=34)
    tr = xm.load_traces(c.bytes, c.tag, c.off)
    assert tr.packed is not None and len(tr.packed) == tr.n_events
    v = tr.packed
    mag = (v & np.uint64((1 << 41) - 1)).astype(np.int64)
    b = np.where((v >> np.uint64(41)) & np.uint64(1), mag, -mag)
    t = ((v >> np.uint64(46)) | (((v >> np.uint64(42)) & np.uint64(0xF)) << np.uint64(28))).astype(np.uint32)
    assert (b == tr.bytes).all() and (t == tr.tag).all()


def test_widened_entry_points_fail_loudly_without_gpu():
    """Every device entry point of the widened rows returns an error (never a
    CPU fallback) when there is no CUDA device."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = xm.lib()
    ins = xm._Instants(None, None, None, None, 1, 0, 0)
    assert L.xm_reconstruct(ctypes.byref(ins), None, 0, None, None, None, None) != 0
    assert L.xm_blocks_from_instants(ctypes.byref(ins), *([None] * 8)) != 0
    prof = xm._Profiles(None, None, None, None, None, None, None, 1, 0, 0)
    assert L.xm_orchestrate(ctypes.byref(prof), 1, None, 0, None, None, None, None) != 0
    m = xm._Metrics()
    assert L.xm_metrics_batch(None, 1, None, 0, ctypes.byref(m), None) != 0


@pytest.mark.parametrize("field,value", [("min_large_alloc", 1 << 20),      # == small_size
                                         ("min_large_alloc", 22 << 20),     # > large_buffer
                                         ("large_buffer", 8 << 20)])        # < min_large_alloc
def test_config_rejects_inconsistent_thresholds(field, value):
    """small_size < min_large_alloc <= large_buffer (torch's
    constants): otherwise a request between them would get a segment smaller
    than itself. Checked before any device work, so testable on CPU."""
    c = hand.h1(512, 3)
    tr = xm.load_traces(c.bytes, c.tag, c.off)
    b = xm._Batch(None, None, None, None, None, None, tr.n_traces, tr.n_events, tr.max_ids,
                  tr.max_events)
    cfg = xm.Config()
    setattr(cfg, field, value)
    cc = cfg.c()
    rc = xm.lib().xm_simulate_batch(ctypes.byref(b), ctypes.byref(cc), None, 0, None, None)
    assert rc == -1, rc                                          # XM_EINVAL
    assert b"min_large_alloc" in xm.lib().xm_last_error()


def test_arena_scratch_is_bounded_for_one_huge_trace():
    """every overflow arena slot is sized for the longest trace, so
    the slot count is capped by a byte budget (4 GiB) instead of one per warp."""
    b = xm._Batch(None, None, None, None, None, None, 5000, 60_000_000, 2_000_000, 50_000_000)
    cc = xm.Config().c()
    n = xm.lib().xm_scratch_bytes(ctypes.byref(b), ctypes.byref(cc))
    per_slot = 50_000_001 * 24 + 2_000_000 * 20
    assert per_slot <= n <= max(4 << 30, per_slot) + (1 << 20)
