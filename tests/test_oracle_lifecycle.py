"""Pins of the lifecycle-reconstruction oracle (oracle/lifecycle.c; SURVEY
NEXT-3; §3.2). No GPU."""
import numpy as np
import pytest

import oracle
from workloads import fuzz, instants, suites


def _rec(addr, by):
    return oracle.reconstruct(np.array(addr, np.uint64), np.array(by, np.int64))


def test_spec_examples():
    # S:109  [+1024@A t=1, -1024@A t=5] -> one block [1,5]
    p, m, t = _rec([0xA, 0xA], [1024, -1024])
    assert p.tolist() == [1, 0] and t["n_blocks"] == 1 and t["n_persistent"] == 0
    # S:110  address reuse after close opens a fresh block; the second is persistent
    p, m, t = _rec([0xA, 0xA, 0xA], [1024, -1024, 2048])
    assert p.tolist() == [1, 0, -1] and t["n_blocks"] == 2 and t["n_persistent"] == 1
    # S:111  a lone free -> zero blocks, orphan tally 1
    p, m, t = _rec([0xB], [-512])
    assert p.tolist() == [-1] and t["n_blocks"] == 0 and t["n_orphan"] == 1


def test_lifo_and_mismatch():
    # two blocks open at one address (a lost free): the free closes the later one (D1)
    p, m, t = _rec([5, 5, 5, 5], [100, 200, -200, -100])
    assert p.tolist() == [3, 2, 1, 0] and t["max_open"] == 2
    # size mismatch: tallied, the block is still closed
    p, m, t = _rec([5, 5], [100, -96])
    assert p.tolist() == [1, 0] and m.tolist() == [0, 1] and t["n_mismatch"] == 1


def brute(addr, by):
    """LIFO per address stated directly: each free takes the latest earlier
    allocation at its address that no earlier free has taken. O(n^2)."""
    n = len(by)
    partner = [-1] * n
    taken = [False] * n
    for i in range(n):
        if by[i] > 0:
            continue
        for j in range(i - 1, -1, -1):
            if by[j] > 0 and addr[j] == addr[i] and not taken[j]:
                taken[j] = True
                partner[i], partner[j] = j, i
                break
    return partner


def _corpus():
    b = fuzz.spec1_corpus(40, 400, salt=31)
    c3 = suites.config3().subset([0, 43])
    c3 = c3.subset([0])
    return [instants.from_batch(b, salt=1, p_orphan=0.01, p_mismatch=0.01, p_lost=0.02),
            instants.from_batch(c3, salt=2, p_orphan=0.002, p_mismatch=0.002, p_lost=0.005)]


def test_bruteforce_and_conservation():
    for ins in _corpus():
        for t in range(ins.n_traces):
            a, by, st = ins.trace(t)
            if len(by) > 3000:
                a, by, st = a[:3000], by[:3000], st[:3000]
            p, m, tal = oracle.reconstruct(a, by)
            assert p.tolist() == brute(a.tolist(), by.tolist())
            # mismatch flags: matched frees whose size differs
            fr = np.flatnonzero((by < 0) & (p >= 0))
            assert (m[fr] == (by[p[fr]] != -by[fr])).all() and m[by > 0].sum() == 0
            # conservation: with no orphans or mismatches the sum of
            # open blocks equals the folded signed stream
            if tal["n_orphan"] == 0 and tal["n_mismatch"] == 0:
                assert int(by[p >= 0].sum()) == 0
            assert tal["n_blocks"] == int((by > 0).sum())
            assert tal["n_orphan"] == int(((by < 0) & (p < 0)).sum())
            assert tal["n_persistent"] == int(((by > 0) & (p < 0)).sum())


def test_clean_trace_roundtrip():
    """Without noise, reconstruction recovers the original trace exactly (the
    wire stream it defines replays to the same result as the id-based trace)."""
    b = suites.config1()
    ins = instants.from_batch(b, salt=3)
    a, by, st = ins.trace(0)
    p, m, tal = oracle.reconstruct(a, by)
    assert tal["n_orphan"] == tal["n_mismatch"] == tal["n_persistent"] == 0
    wb, wt, kept = oracle.wire_from_partner(by, st, p)
    ob, ot = b.trace(0)
    assert (wb == ob).all()
    r1, _ = oracle.simulate_trace(wb, wt)
    r2, _ = oracle.simulate_trace(ob, ot)
    assert r1 == r2
