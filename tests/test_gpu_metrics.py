"""NEXT-4 batched metrics on the GPU (xm_metrics_batch) vs oracle/metrics.py,
exact (fp64 with the same operation order on both sides). Runs are seeded
synthetic records; the estimates of one set come from an actual config-5
replay (peak_reserved, Eq. 1), the 'measurements' are synthetic."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2510_21048_b200 as xm
from oracle import metrics as OM

GiB = 1 << 30


def _records(n, seed, est=None, m_max=None):
    rng = np.random.default_rng(seed)
    r = np.zeros(n, xm.RUN_DTYPE)
    r["m_max"] = m_max if m_max is not None else rng.choice([8 * GiB, 12 * GiB, 40 * GiB], n)
    r["m_peak_est"] = est if est is not None else rng.integers(1, 2 * r["m_max"].astype(np.int64))
    r["oom_pred"] = r["m_peak_est"] > r["m_max"]
    r["oom1"] = rng.random(n) < 0.3
    c1 = r["oom_pred"] == r["oom1"]
    run2 = c1 & (r["oom1"] == 0)
    r["oom2"] = np.where(run2, rng.random(n) < 0.2, xm.ROUND2_NOT_RUN)
    r["m_peak_meas1"] = rng.integers(1, r["m_max"].astype(np.int64))
    r["m_peak_meas2"] = rng.integers(1, r["m_max"].astype(np.int64))
    return r


def _oracle(r):
    runs = [dict(est=int(x["m_peak_est"]), meas1=int(x["m_peak_meas1"]), meas2=int(x["m_peak_meas2"]),
                 m_max=int(x["m_max"]), oom_pred=bool(x["oom_pred"]), oom1=bool(x["oom1"]),
                 oom2=None if x["oom2"] == xm.ROUND2_NOT_RUN else bool(x["oom2"])) for x in r]
    return OM.evaluate(runs)


def _same(g, o):
    for k in ("n", "n_mre", "sum_c1", "sum_c2", "sum_save"):
        assert g[k] == o[k], k
    for k in ("mre", "pef1", "pef2", "mcp"):
        assert (math.isnan(g[k]) and math.isnan(o[k])) or g[k] == o[k], (k, g[k], o[k])


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 1), (7, 2), (1000, 3), (20001, 4)])
def test_metrics_random_records(n, seed):
    r = _records(n, seed)
    _same(xm.metrics(r), _oracle(r))


def test_metrics_from_a_replay():
    from workloads import mc5
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    idx = np.arange(0, 40000, 7)
    d = mc5.describe(idx)
    pool = xm.Templates(*mc5.template_pool())
    dev = xm.expand_templates(pool, d["tpl"], d["b"], d["seed"], mc5.SWAP_THRESHOLD)  # unlimited
    h, _ = xm.peaks(xm.simulate_batch(dev))
    r = _records(len(idx), 5, est=h["peak_reserved"].astype(np.uint64), m_max=d["capacity"])
    _same(xm.metrics(r), _oracle(r))


def test_metrics_errors():
    with pytest.raises(xm.XMemError):
        xm.metrics(np.zeros(0, xm.RUN_DTYPE))
    r = _records(10, 6)
    bad = r.copy()
    k = int(np.flatnonzero(bad["oom_pred"] != bad["oom1"])[0])   # C1 = 0 ...
    bad["oom2"][k] = 0                                            # ... but a round 2
    with pytest.raises(xm.XMemError):
        xm.metrics(bad)
