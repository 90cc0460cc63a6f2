"""Config 5 (BASELINE configs[4], Monte Carlo at paper scale):
traces expanded ON THE DEVICE by K4 (xm_expand_templates) equal the host
recipe (workloads/mc5.py) byte for byte, and their replay equals the oracle
bit-exactly -- on a few thousand traces in full, and at the full 1M-trace size
(the bench's launch configuration) on a sample the oracle replays one by one."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2510_21048_b200 as xm
import oracle_pool
from gpu_util import assert_parity, oracle_run
from workloads import mc5


@pytest.fixture(scope="module")
def pool():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    f, p, t, off, nids = mc5.template_pool()
    return xm.Templates(f, p, t, off, nids)


def _expand(pool, idx):
    d = mc5.describe(idx)
    dev = xm.expand_templates(pool, d["tpl"], d["b"], d["seed"], mc5.SWAP_THRESHOLD,
                              capacity=d["capacity"])
    return dev, d


def test_expand_matches_host_recipe(pool):
    idx = np.arange(0, 3_000_000, 1013)[:2500]
    dev, _ = _expand(pool, idx)
    host = mc5.batch(idx)
    by = dev.bytes.cpu().numpy()
    tg = dev.tag.cpu().numpy().view(np.uint32)
    off = dev.off.cpu().numpy()
    order = dev.order.cpu().numpy().view(np.uint32)
    for k in range(len(idx)):
        t = int(order[k])
        hb, ht = host.trace(t)
        assert (by[off[k]:off[k + 1]] == hb).all(), t
        assert (tg[off[k]:off[k + 1]] == ht).all(), t


def test_expanded_batch_replay_parity(pool):
    idx = np.arange(7, 7 + 3000 * 331, 331)
    dev, _ = _expand(pool, idx)
    res = xm.simulate_batch(dev)
    h, summ = xm.peaks(res)
    assert summ["n_overflow"] == 0
    assert_parity(mc5.batch(idx), h, oracle_run(mc5.batch(idx), parallel=True))


def test_full_size_one_million_traces(pool):
    """1M traces (~5.6e9 events, ~68 GB) expanded and replayed in the bench's
    launch configuration; parity vs the oracle on a >= 300k-trace slice that
    holds every simulated OOM, the 1000 longest traces and every 5th trace,
    each rebuilt on the host independently of K4 (workloads/mc5gen.c) and
    replayed by the oracle on all host cores. (bench.py --workload cfg5
    compares all 1M.)"""
    n = 1_000_000
    if torch.cuda.get_device_properties(0).total_memory < (100 << 30):
        pytest.skip("needs a 180 GB B200")
    idx = np.arange(n)
    dev, d = _expand(pool, idx)
    res = xm.simulate_batch(dev)
    h, summ = xm.peaks(res)
    del dev, res
    torch.cuda.empty_cache()
    assert summ["n_overflow"] == 0 and summ["n_traces"] == n
    L = mc5.lengths(d)
    assert summ["events_done"] <= int(L.sum())
    oom = np.flatnonzero(h["status"] == 1)
    assert len(oom) > 1000
    sample = np.unique(np.r_[oom, np.argsort(-L, kind="stable")[:1000], np.arange(0, n, 5)])
    assert len(sample) >= 100_000
    s = oracle_pool.parity_mc5(sample, h)
    assert s["traces"] == len(sample)
    assert s["mismatched_values"] == 0, s
    assert s["oracle_oom_traces"] == len(oom)          # every OOM trace is in the sample
