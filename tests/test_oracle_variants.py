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
