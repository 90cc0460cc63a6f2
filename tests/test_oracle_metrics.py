"""Pins of oracle/metrics.py (NEXT-4 batched metrics) to SPEC.md's worked
examples and to properties of the paper's equations
(PAPER.md:445-481). No GPU."""
import math
import random

import pytest

from oracle import metrics as M

GiB = 1 << 30


@pytest.mark.parametrize("est,meas,exp", [(110, 100, 0.10), (100, 100, 0.0), (50, 100, 0.50)])
def test_relative_error_examples(est, meas, exp):
    assert M.relative_error(est, meas) == pytest.approx(exp, abs=0, rel=1e-15)


def test_relative_error_undefined():
    with pytest.raises(M.MetricsError):
        M.relative_error(5, 0)


def test_median_examples():
    assert M.median([0.1, 0.3, 0.2]) == 0.2
    assert M.median([0.1, 0.3]) == (0.1 + 0.3) / 2
    assert M.median([0.07]) == 0.07


def test_correctness_examples():
    assert M.correctness1(True, True) == 1 and M.correctness1(False, True) == 0
    assert M.correctness1(False, False) == 1
    assert M.correctness2(1, False, False) == 1 and M.correctness2(1, True, False) == 0
    assert M.correctness2(1, None, True) == 1


def _run(est, m_max, oom_pred, oom1, oom2, meas1=1, meas2=1):
    return dict(est=est, m_max=m_max, oom_pred=oom_pred, oom1=oom1, oom2=oom2, meas1=meas1,
                meas2=meas2)


def test_pef_example():                                  # C2 = {1,1,0,1} -> 0.25
    runs = [_run(1, 10, False, False, False), _run(1, 10, False, False, False),
            _run(1, 10, False, False, True), _run(1, 10, False, False, False)]
    r = M.evaluate(runs)
    assert r["pef2"] == 0.25 and r["pef1"] == 0.0


def test_memory_saving_examples():
    assert M.memory_saving(1, False, False, 8 * GiB, 12 * GiB) == 4 * GiB
    assert M.memory_saving(1, True, None, 20 * GiB, 12 * GiB) == 12 * GiB
    assert M.memory_saving(0, False, None, 8 * GiB, 12 * GiB) == -12 * GiB


def test_mcp_example():                                  # {+4, -12} GiB -> -4 GiB
    runs = [_run(8 * GiB, 12 * GiB, False, False, False),      # C1=1, OOM2=0: +4
            _run(8 * GiB, 12 * GiB, True, False, None)]        # C1=0: -12
    assert M.evaluate(runs)["mcp"] == -4 * GiB


def test_gating_rejected():                              # SPEC D2
    with pytest.raises(M.MetricsError):
        M.evaluate([_run(1, 10, True, False, False)])    # C1=0 but round 2 present


def _random_runs(n, seed):
    rng = random.Random(seed)
    runs = []
    for _ in range(n):
        m_max = rng.choice([8 * GiB, 12 * GiB, 40 * GiB])
        est = rng.randint(1, 2 * m_max)
        oom_pred = est > m_max                                   # Eq. 1
        oom1 = rng.random() < 0.3
        c1 = oom_pred == oom1
        oom2 = (rng.random() < 0.2) if (c1 and not oom1) else None
        runs.append(_run(est, m_max, oom_pred, oom1, oom2, rng.randint(1, m_max), rng.randint(1, m_max)))
    return runs


def test_properties():
    runs = _random_runs(501, 3)
    r = M.evaluate(runs)
    shuffled = runs[:]
    random.Random(9).shuffle(shuffled)
    assert M.evaluate(shuffled) == r                     # permutation invariance
    c2 = [M.correctness2(M.correctness1(x["oom_pred"], x["oom1"]), x["oom2"], x["oom1"]) for x in runs]
    assert r["pef2"] == pytest.approx(1 - sum(c2) / len(c2), abs=1e-15)
    assert 0 <= r["pef1"] <= 1 and 0 <= r["pef2"] <= 1 and r["mre"] >= 0
    assert r["pef2"] >= r["pef1"]                        # C2 implies C1
    # a run with C1 = 0 contributes exactly -M_max
    bad = [x for x in runs if M.correctness1(x["oom_pred"], x["oom1"]) == 0]
    assert all(M.memory_saving(0, x["oom1"], x["oom2"], x["est"], x["m_max"]) == -x["m_max"]
               for x in bad)
    # MRE is the middle order statistic of the selected errors
    errs = sorted(M.relative_error(x["est"], x["meas2"] if x["oom2"] is False else x["meas1"])
                  for x in runs if not x["oom1"])
    assert len(errs) == r["n_mre"]
    k = len(errs)
    assert r["mre"] == (errs[k // 2] if k % 2 else (errs[k // 2 - 1] + errs[k // 2]) / 2)
    assert math.isnan(M.evaluate([_run(5, 4, True, True, None)])["mre"])
