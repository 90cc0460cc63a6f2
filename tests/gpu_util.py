"""Helpers for -m gpu parity tests: run the CUDA path through the C-ABI and
compare every result field with the oracle, element by element, bit-exact."""
import numpy as np

import oracle
import paper_2510_21048_b200 as xm

# fields compared (the oracle has the same names; n_free_blocks_end saturates at 65535)
COMPARE = ["peak_allocated", "peak_allocated_idx", "peak_allocated_blk", "peak_allocated_blk_idx",
           "peak_reserved", "peak_reserved_idx", "final_reserved", "n_seg_alloc",
           "n_seg_release", "max_live_segments", "events_done", "status", "n_free_blocks_end"]


def gpu_run(batch, cfg=None, capacity=True):
    cfg = cfg or xm.Config()
    tr = xm.load_traces(batch.bytes, batch.tag, batch.off)
    cap = batch.capacity if capacity and (batch.capacity != oracle.UNLIMITED).any() else None
    dev = tr.to_device(capacity=cap)
    res = xm.simulate_batch(dev, cfg)
    h, summ = xm.peaks(res)
    return h, summ


def oracle_run(batch, strict=1, parallel=False, div=0, reclaim=0, msplit=None, gc=0.0):
    ocfg = oracle.Config(large_split_strict=strict, roundup_power2_divisions=div,
                         reclaim_policy=reclaim, gc_threshold=gc,
                         **({"max_split_size": msplit} if msplit is not None else {}))
    if parallel:
        import oracle_pool
        return oracle_pool.run(batch, ocfg)
    return oracle.simulate_batch(batch, ocfg)


def assert_parity(batch, h, o, fields=COMPARE, mode_full=True):
    T = batch.n_traces
    assert h.shape[0] == T
    for f in fields:
        exp = o[f].astype(np.uint64)
        if f == "n_free_blocks_end":
            exp = np.minimum(exp, 65535)
        got = h[f].astype(np.uint64)
        bad = np.flatnonzero(got != exp)
        if len(bad):
            t = int(bad[0])
            name = batch.names[t] if batch.names else t
            raise AssertionError(f"field {f}: {len(bad)}/{T} traces differ; first trace {t} "
                                 f"({name}): gpu={int(got[t])} oracle={int(exp[t])}")
