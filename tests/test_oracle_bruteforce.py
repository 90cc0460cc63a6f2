"""Oracle vs the independent gap-model brute force (tests/bruteforce.py).

SPEC.md:508 acceptance #1: seeded random sequences (<= 1,000 events, sizes
1 B - 64 MiB) must give identical (allocated, reserved) timelines, zero
tolerance. Here every per-event curve value and every result field is
compared, on all 1,000 sequences (about 5 s).
"""
import numpy as np
import pytest

import bruteforce
import oracle
from workloads import fuzz, hand

N_SPEC1 = 1000


def _compare(batch, strict=True):
    cfg = oracle.Config(large_split_strict=int(strict))
    for t in range(batch.n_traces):
        by, tg = batch.trace(t)
        cap = int(batch.capacity[t])
        o, oc = oracle.simulate_trace(by, tg, cap, cfg=cfg, curve=True)
        b, bc = bruteforce.simulate(by, tg, cap, strict=strict)
        for k, v in b.items():
            assert o[k] == v, (batch.names[t] if batch.names else t, k, o[k], v)
        n = o["events_done"]
        assert oc[:n].tolist() == [list(x) for x in bc[:n]], t


def test_spec1_corpus():
    _compare(fuzz.spec1_corpus(N_SPEC1, 1000, salt=1))


def test_small_pool_corpus():
    _compare(fuzz.small_size_corpus(150, 400, salt=2))


def test_capacity_corpus():
    c = fuzz.capacity_corpus(150, 500, salt=3)
    _compare(c)
    r = oracle.simulate_batch(c)
    assert (r["status"] == 1).sum() > 10 and (r["n_seg_release"] > 0).sum() > 10


def test_spec_split_variant():
    _compare(fuzz.spec1_corpus(60, 400, salt=4), strict=False)


def test_fragmentation_stress():
    _compare(fuzz.fragmentation_stress())


def test_hand_traces_bruteforce(golden):
    """The goldens hold for the brute force too (pins the brute force)."""
    tr = hand.all_named()
    for name, g in golden.items():
        b = tr[name]
        res, _ = bruteforce.simulate(b.bytes, b.tag, int(b.capacity[0]))
        for k, v in g["expect"].items():
            assert res[k] == v, (name, k)
