"""The host-parallel oracle harness (tests/oracle_pool.py) used by bench.py's
cpu_baseline / reference arm and by the full-size config-5 parity: same
results as the single-process oracle, and the parity counter catches a
perturbed field. No GPU."""
import numpy as np

import oracle
import oracle_pool
import paper_2510_21048_b200 as xm
from workloads import fuzz, mc5


def test_pool_equals_single_process():
    b = fuzz.capacity_corpus(60, 300, salt=71)
    ref = oracle.simulate_batch(b)
    with oracle_pool.Pool(b, workers=3) as p:
        for _ in range(2):                          # reusable across passes
            got, wall, busiest, total = p.run()
            for k in oracle.FIELDS:
                assert (got[k] == ref[k]).all(), k
            assert 0 < busiest <= total


def _as_results(o, T):
    h = np.zeros(T, xm.RESULT_DTYPE)
    for k in xm.FIELDS:
        h[k] = o[k].astype(h[k].dtype) if k != "n_free_blocks_end" else np.minimum(o[k], 65535)
    return h


def test_mc5_parity_counts_mismatches():
    idx = np.arange(3000, 3000 + 900, 3)
    o = oracle.simulate_batch(mc5.batch(idx))
    h = _as_results(o, len(idx))
    s = oracle_pool.parity_mc5(idx, h, pos=np.arange(len(idx)), workers=2, chunk_traces=70)
    assert s["traces"] == len(idx) and s["mismatched_values"] == 0
    assert s["oracle_events"] == int(o["events_done"].sum())
    h["peak_reserved"][17] += 512
    h["status"][250] ^= 1
    s = oracle_pool.parity_mc5(idx, h, pos=np.arange(len(idx)), workers=2, chunk_traces=70)
    assert s["mismatched_values"] == 2
    assert s["first_mismatch_trace"] == int(idx[17])
    assert set(s["mismatched_by_field"]) == {"peak_reserved", "status"}
