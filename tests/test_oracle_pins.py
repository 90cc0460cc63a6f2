"""Pins of the oracle to the paper, SPEC.md and closed forms (no GPU).

Each assertion checks oracle/ against something other than itself: worked
examples printed in SPEC.md/PAPER.md, hand-derived closed forms (goldens with
citations in tests/golden/hand_traces.json), and invariants.
"""
import numpy as np
import pytest

import oracle
from workloads import hand
from workloads.trace import TraceBuilder

MiB = 1 << 20


# ---- a2: round-up (PAPER.md:153-154, 256 (i)) -------------
@pytest.mark.parametrize("req,exp", [(1, 512), (512, 512), (513, 1024), (1023, 1024),
                                     (1024, 1024), (10**6, 1000448), (10**7, 10000384)])
def test_round_size_examples(req, exp):
    assert oracle.round_size(req) == exp


def test_round_size_closed_form_random():
    rng = np.random.default_rng(0)
    for req in rng.integers(1, 1 << 40, 2000):
        s = oracle.round_size(int(req))
        assert s % 512 == 0 and s >= req and s - req < 512


# ---- a4: pool + segment size (PAPER.md:169, 257 (ii), 654) --
@pytest.mark.parametrize("s,exp", [(512, 2 * MiB), (MiB, 2 * MiB), (MiB + 512, 20 * MiB),
                                   (2 * MiB, 20 * MiB), (10 * MiB - 512, 20 * MiB),
                                   (10 * MiB, 10 * MiB), (11 * MiB, 12 * MiB),
                                   (78 * MiB, 78 * MiB), (19 * MiB, 20 * MiB)])
def test_segment_size_examples(s, exp):
    assert oracle.segment_size(s) == exp


def test_pool_threshold():
    assert oracle.is_small(MiB) and not oracle.is_small(MiB + 512)


# ---- a7: split rule (reading Q1) -------------------------------
def test_split_rule():
    assert oracle.should_split(True, 512) and not oracle.should_split(True, 0)
    assert not oracle.should_split(False, MiB)          # torch strict
    assert oracle.should_split(False, MiB + 512)
    assert oracle.should_split(False, MiB, oracle.Config(large_split_strict=0))  # SPEC >=


# ---- goldens: hand traces with cited expected values -------------------------
def test_hand_goldens(golden):
    traces = hand.all_named()
    assert set(golden) <= set(traces)
    for name, g in golden.items():
        b = traces[name]
        res, curve = oracle.simulate_trace(b.bytes, b.tag, int(b.capacity[0]), curve=True,
                                           check=True)
        for k, v in g["expect"].items():
            assert res[k] == v, (name, k, res[k], v, g["cite"])
        if "curve" in g:
            assert curve.tolist() == g["curve"], name


def test_h6_spec_split_variant():
    b = hand.h6()
    res, _ = oracle.simulate_trace(b.bytes, b.tag, cfg=oracle.Config(large_split_strict=0))
    assert res["peak_allocated_blk"] == 19 * MiB   # SPEC.md:248 '>=' reading


# ---- Eq. 1 -------------------------------
def test_eq1_strict():
    G = 1 << 30
    # capacity == exact peak -> fits (strict >); one byte less -> OOM
    b = TraceBuilder().alloc(0, 12 * G).end_trace().build()
    fits, _ = oracle.simulate_trace(b.bytes, b.tag, capacity=12 * G)
    oom, _ = oracle.simulate_trace(b.bytes, b.tag, capacity=12 * G - 1)
    assert fits["status"] == 0 and fits["peak_reserved"] == 12 * G
    assert oom["status"] == 1 and oom["events_done"] == 0


# ---- contract violations -----------------------------
def _raw(ev):
    by = np.array([e[0] for e in ev], np.int64)
    tg = np.array([e[1] for e in ev], np.uint32)
    return by, tg


@pytest.mark.parametrize("ev,code", [([(0, 1)], -1),
                                     ([(512, 1), (512, 1)], -2),
                                     ([(-512, 1)], -3),
                                     ([(512, 1), (-1024, 1)], -4)])
def test_contract_violations(ev, code):
    by, tg = _raw(ev)
    with pytest.raises(oracle.OracleError) as e:
        oracle.simulate_trace(by, tg)
    assert e.value.code == code


# ---- invariants after every event --------------------------
def test_invariants_fuzz():
    from workloads import fuzz
    for salt, corpus in ((11, fuzz.spec1_corpus(60, 400, salt=11)),
                         (12, fuzz.small_size_corpus(60, 300, salt=12)),
                         (13, fuzz.capacity_corpus(60, 300, salt=13))):
        r = oracle.simulate_batch(corpus, check=True)   # raises on any violation
        assert (r["peak_allocated"] <= r["peak_allocated_blk"]).all()
        assert (r["peak_allocated_blk"] <= r["peak_reserved"]).all()
        assert (r["peak_reserved"] <= corpus.capacity).all()
        assert (r["peak_reserved"] % (2 * MiB) == 0).all()
        closed = r["status"] == 0
        assert (r["final_allocated"][closed] == 0).all()
        # closed trace: every live segment is one free block (coalescing maximality)
        live = r["n_seg_alloc"] - r["n_seg_release"]
        assert (r["n_free_blocks_end"][closed] == live[closed]).all()


def test_determinism():
    from workloads import fuzz
    c = fuzz.spec1_corpus(20, 300, salt=5)
    a = oracle.simulate_batch(c)
    b = oracle.simulate_batch(c)
    for k in a:
        assert (a[k] == b[k]).all()


def test_peak_allocated_is_max_prefix_sum():
    """peak_allocated = max prefix sum of +-round512 (brute force O(n))."""
    from workloads import fuzz
    c = fuzz.spec1_corpus(40, 500, salt=7)
    r = oracle.simulate_batch(c)
    for t in range(c.n_traces):
        by, _ = c.trace(t)
        d = np.sign(by) * (((np.abs(by) + 511) // 512) * 512)
        ps = np.cumsum(d)
        assert r["peak_allocated"][t] == ps.max()
        assert r["peak_allocated_idx"][t] == int(np.argmax(ps))


def test_sequence_sensitivity_tally():
    """Reading Q11: SPEC.md:510 '#3 late >= early' is not an invariant of BFC; H3
    is the constructed counterexample and H4 the Fig. 2 witness (strict >)."""
    n = hand.all_named()
    r = {k: oracle.simulate_trace(n[k].bytes, n[k].tag)[0]["peak_reserved"]
         for k in ("H3-early", "H3-late", "H4-early", "H4-late")}
    assert r["H3-early"] > r["H3-late"]
    assert r["H4-late"] > r["H4-early"]
