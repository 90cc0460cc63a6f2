"""allocator variants in the oracle, pinned (no GPU).

* roundup_power2_divisions:N -- PyTorch's PYTORCH_CUDA_ALLOC_CONF knob the paper's
  simulator would need for jobs that set it (PAPER.md:257 defers to the PyTorch
  allocator; reading Q15/Q20). Pinned by hand-computed values from its
  definition (N equal steps between consecutive powers of two), by an
  independent brute force, and on the box by the real allocator
  (tests/test_torch_allocator_pin.py).
* reclaim_policy=1 -- SPEC.md:283 D3 "Reclamation releases only fully-free
  segments, both pools, largest first, stopping when capacity suffices"
  (reading Q19: ties by lowest address). Pinned by the hand trace H8 and the
  brute force.
"""
import pytest

import bruteforce
import oracle
from workloads import fuzz, hand

MiB = 1 << 20
GiB = 1 << 30


@pytest.mark.parametrize("div,req,exp", [
    (4, 1_000_000, MiB),                  # [512 KiB, 1 MiB) in steps of 128 KiB
    (4, 3 * MiB // 2 + 1, 7 * MiB // 4),  # [1, 2) MiB in steps of 256 KiB
    (4, 2 * MiB, 2 * MiB),                # a power of two stays
    (4, 2000, 2048),                      # <= 512 * 4: plain 512 B rounding
    (4, 600, 1024),                       # (not 640 = the next 128 B step)
    (8, 3000, 3072),                      # <= 512 * 8
    (4, 2048, 2048),
    (4, 2049, 2560),                      # [2048, 4096) in steps of 512
    (4, 3000, 3072),
    (4, 5 * GiB, 5 * GiB),                # on a step of [4, 8) GiB
    (4, 5 * GiB + 1, 6 * GiB),
    (2, 3 * MiB + 1, 4 * MiB),            # [2, 4) MiB in steps of 1 MiB
    (8, 9 * MiB + 1, 10 * MiB),           # [8, 16) MiB in steps of 1 MiB
    (1, 1_000_000, 1000448),              # 1 division = off
    (0, 1_000_000, 1000448),
])
def test_roundup_power2_divisions_values(div, req, exp):
    assert oracle.round_size(req, oracle.Config(roundup_power2_divisions=div)) == exp
    assert bruteforce.rnd(req, div=div) == exp


def test_roundup_changes_pool_choice():
    # 1,000,000 B rounds to exactly 1 MiB: still the small pool (s <= 1 MiB)
    c = oracle.Config(roundup_power2_divisions=4)
    assert oracle.is_small(oracle.round_size(1_000_000, c), c)
    assert not oracle.is_small(oracle.round_size(MiB + 1, c), c)


def _compare(batch, div=0, reclaim=0):
    cfg = oracle.Config(roundup_power2_divisions=div, reclaim_policy=reclaim)
    for t in range(batch.n_traces):
        by, tg = batch.trace(t)
        cap = int(batch.capacity[t])
        o, oc = oracle.simulate_trace(by, tg, cap, cfg=cfg, curve=True, check=True)
        b, bc = bruteforce.simulate(by, tg, cap, div=div, reclaim=reclaim)
        for k, v in b.items():
            assert o[k] == v, (t, k, o[k], v)
        n = o["events_done"]
        assert oc[:n].tolist() == [list(x) for x in bc[:n]], t


@pytest.mark.parametrize("div", [2, 4, 8])
def test_roundup_vs_bruteforce(div):
    _compare(fuzz.spec1_corpus(150, 500, salt=60 + div), div=div)
    _compare(fuzz.small_size_corpus(60, 400, salt=70 + div), div=div)


def test_d3_reclaim_vs_bruteforce():
    c = fuzz.capacity_corpus(200, 500, salt=81)
    _compare(c, reclaim=1)
    r0 = oracle.simulate_batch(c)
    r1 = oracle.simulate_batch(c, oracle.Config(reclaim_policy=1))
    # the two policies do lead to different replays on this corpus
    assert (r1["n_seg_release"] != r0["n_seg_release"]).any()
    _compare(c, div=4, reclaim=1)


def test_h8_release_all_vs_largest_first():
    b = hand.h8()
    by, tg = b.trace(0)
    t, _ = oracle.simulate_trace(by, tg, 32 * MiB)
    d, _ = oracle.simulate_trace(by, tg, 32 * MiB, cfg=oracle.Config(reclaim_policy=1))
    # torch: both cached segments go, then the 12 MiB segment (reading Q3)
    assert (t["n_seg_release"], t["final_reserved"], t["peak_reserved"]) == (2, 12 * MiB, 22 * MiB)
    # SPEC D3: only the 20 MiB one (2 + 12 <= 32 after it), then the 12 MiB segment
    assert (d["n_seg_release"], d["final_reserved"], d["peak_reserved"]) == (1, 14 * MiB, 22 * MiB)
    assert t["status"] == d["status"] == 0


# ---- torch max_split_size_mb / garbage_collection_threshold (readings Q26, Q27) --
def _knobs(by, tg, cap, msplit=None, gc=0.0):
    kw = {}
    if msplit is not None:
        kw["max_split_size"] = msplit
    o, _ = oracle.simulate_trace(by, tg, cap, cfg=oracle.Config(gc_threshold=gc, **kw), check=True)
    b, _ = bruteforce.simulate(by, tg, cap, msplit=msplit, gc=gc)
    for k, v in b.items():
        assert o[k] == v, (k, o[k], v)
    return o


def _one(build, cap=oracle.UNLIMITED):
    from workloads.trace import TraceBuilder
    tb = TraceBuilder()
    build(tb)
    tb.end_trace(capacity=cap)
    return tb.build().trace(0)


def test_h9_max_split_size_no_split_no_oversize_reuse():
    """max_split_size_mb:64. A 100 MiB request gets a 100 MiB segment and is
    never split; a 90 MiB request reuses the cached 100 MiB block whole (100 <
    90 + 20 MiB); a 30 MiB request may not take a block of >= 64 MiB, and a
    70 MiB one not a block of >= 70 + 20 MiB: both get new segments.
    Reserved 100 + 30 + 70 = 200 MiB; without the knob the 100 MiB segment
    serves everything (100 MiB)."""
    by, tg = _one(lambda t: t.alloc(0, 100 * MiB).free(0).alloc(1, 90 * MiB).free(1)
                  .alloc(2, 30 * MiB).alloc(3, 70 * MiB))
    o = _knobs(by, tg, oracle.UNLIMITED, msplit=64 * MiB)
    assert (o["peak_reserved"], o["n_seg_alloc"], o["peak_allocated_blk"]) == (200 * MiB, 3, 100 * MiB)
    assert o["peak_allocated_blk_idx"] == 0           # B (90 MiB) holds the whole 100 MiB block
    o0 = _knobs(by, tg, oracle.UNLIMITED)
    assert (o0["peak_reserved"], o0["n_seg_alloc"]) == (100 * MiB, 1)


def test_h10_release_available_releases_one_fitting_block():
    """max_split_size_mb:64, capacity 180 MiB. Cached: 100 MiB, 30 MiB and a
    2 MiB small segment (132 MiB). A 70 MiB request may not reuse the 100 MiB
    block (>= 70 + 20 MiB), and 132 + 70 > 180: release_available_cached_blocks
    releases just the smallest block >= max(70, 64) MiB = the 100 MiB one,
    then the request fits (32 + 70 = 102 MiB). torch's release-all would also
    drop the 30 and 2 MiB segments."""
    by, tg = _one(lambda t: t.alloc(0, 100 * MiB).alloc(1, 30 * MiB).alloc(2, MiB).free(0).free(1)
                  .free(2).alloc(3, 70 * MiB), 180 * MiB)
    o = _knobs(by, tg, 180 * MiB, msplit=64 * MiB)
    assert (o["n_seg_release"], o["final_reserved"], o["status"]) == (1, 102 * MiB, 0)


def test_h11_release_available_walks_down_from_the_largest():
    """max_split_size_mb:64, capacity 200 MiB. Cached whole segments 66, 70 and
    30 MiB (166). A 120 MiB request: no block >= 120 MiB, so oversize blocks
    are released from the largest down until >= 120 MiB are freed: 70, then
    66 (136 >= 120); the 30 MiB one stays (30 + 120 = 150 MiB). With 150 MiB
    requested instead, 70 + 66 = 136 < 150: the walk fails and torch falls
    through to release_cached, which drops the 30 MiB segment as well."""
    by, tg = _one(lambda t: t.alloc(0, 66 * MiB).alloc(1, 70 * MiB).alloc(2, 30 * MiB).free(0)
                  .free(1).free(2).alloc(3, 120 * MiB), 200 * MiB)
    o = _knobs(by, tg, 200 * MiB, msplit=64 * MiB)
    assert (o["n_seg_release"], o["final_reserved"]) == (2, 150 * MiB)
    by, tg = _one(lambda t: t.alloc(0, 66 * MiB).alloc(1, 70 * MiB).alloc(2, 30 * MiB).free(0)
                  .free(1).free(2).alloc(3, 150 * MiB), 200 * MiB)
    o = _knobs(by, tg, 200 * MiB, msplit=64 * MiB)
    assert (o["n_seg_release"], o["final_reserved"]) == (3, 150 * MiB)


def test_h12_garbage_collection_releases_old_cached_segments():
    """garbage_collection_threshold:0.5, capacity 1000 MiB (GC bar 500 MiB).
    Segments 200, 150, 120, 60 MiB (530 MiB; every request so far was a miss:
    4 large-pool searches). Free 200 and 120 (both enter the cache at search
    4). 110 and 100 MiB requests (searches 5 and 6) reuse the 120 MiB block
    and free it again (re-entering at 6). A 300 MiB request (search 7) misses:
    reserved 530 > 500, so GC runs: ages 3 (the 200) and 1 (the 120), mean 2,
    the 200 MiB segment goes (reclaimed 200 >= the 30 MiB excess). Reserved
    330 + 300 = 630 MiB instead of 830."""
    by, tg = _one(lambda t: t.alloc(0, 200 * MiB).alloc(1, 150 * MiB).alloc(2, 120 * MiB)
                  .alloc(3, 60 * MiB).free(0).free(2).alloc(4, 110 * MiB).free(4)
                  .alloc(5, 100 * MiB).free(5).alloc(6, 300 * MiB), 1000 * MiB)
    o = _knobs(by, tg, 1000 * MiB, gc=0.5)
    assert (o["peak_reserved"], o["n_seg_release"]) == (630 * MiB, 1)
    o0 = _knobs(by, tg, 1000 * MiB)
    assert (o0["peak_reserved"], o0["n_seg_release"]) == (830 * MiB, 0)
    # unlimited capacity: no set_fraction, so no GC (torch)
    o1 = _knobs(by, tg, oracle.UNLIMITED, gc=0.5)
    assert o1["peak_reserved"] == 830 * MiB


def _compare_knobs(batch, msplit=None, gc=0.0):
    for t in range(batch.n_traces):
        by, tg = batch.trace(t)
        _knobs(by, tg, int(batch.capacity[t]), msplit=msplit, gc=gc)


@pytest.mark.parametrize("msplit", [21 * MiB, 32 * MiB])
def test_max_split_size_vs_bruteforce(msplit):
    _compare_knobs(fuzz.spec1_corpus(120, 400, salt=90), msplit=msplit)
    _compare_knobs(fuzz.capacity_corpus(150, 500, salt=91), msplit=msplit)


@pytest.mark.parametrize("gc", [0.3, 0.6, 0.9])
def test_garbage_collection_vs_bruteforce(gc):
    _compare_knobs(fuzz.capacity_corpus(150, 500, salt=92), gc=gc)


def test_both_knobs_vs_bruteforce():
    c = fuzz.capacity_corpus(150, 500, salt=93)
    _compare_knobs(c, msplit=24 * MiB, gc=0.5)
    r0 = oracle.simulate_batch(c)
    r1 = oracle.simulate_batch(c, oracle.Config(max_split_size=24 * MiB, gc_threshold=0.5))
    assert (r1["n_seg_release"] != r0["n_seg_release"]).any()
    assert (r1["peak_reserved"] != r0["peak_reserved"]).any()
