"""ORACLE -- test infrastructure only (see oracle/__init__.py).

The paper's evaluation metrics over recorded runs, written out from PAPER.md
§4.1.5 (Eqs. relative-error, median-error, 1st/2nd correctness,
failed-estimation-probability, memory-savings, estimator-memory-average-saving;
PAPER.md:445-481) and SPEC.md's metrics module, for the
NEXT-4 batched-metrics row. Plain Python loops over the runs.

A run is a dict with keys est (M̂peak_jde), meas1 (Mpeak_jd1), meas2
(Mpeak_jd2), m_max (M_d^max), oom_pred (ÔOM_jde, Eq. 1), oom1 (OOM_jd1), oom2
(OOM_jde2: 0, 1, or None = round 2 not run). Floating point is fp64 with one
fixed operation order (integers are converted to float once, then divided),
which the CUDA path follows too.

Readings (Q21): MRE selects runs with OOM_jd1 = 0 and uses
error_jde2 when OOM_jde2 = 0, else error_jde1 (Eq. median-error; a run whose
round 2 was not run counts as OOM_jde2 != 0); the even-count median is the
mean of the central pair (SPEC D1); a record with round-2 fields although
not C1 = 1 and OOM_jd1 = 0 is invalid (SPEC D2, P:385 gating). M_save's
OOM penalty is the equation's -M_max ("-M_max
otherwise"), not P:439's prose "the M̂peak ... is deducted" (Q21).

Parity status: pinned (tests/test_oracle_metrics.py: SPEC.md worked examples
and properties).
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional


class MetricsError(ValueError):
    pass


def relative_error(est: int, meas: int) -> float:
    """Eq. relative-error: |M̂ - M| / M."""
    if meas <= 0:
        raise MetricsError("measured peak must be > 0")
    return float(abs(int(est) - int(meas))) / float(meas)


def correctness1(oom_pred: bool, oom1: bool) -> int:
    """Eq. 1st-correctness: C1 = [ÔOM = OOM_jd1]."""
    return int(bool(oom_pred) == bool(oom1))


def correctness2(c1: int, oom2: Optional[bool], oom1: bool) -> int:
    """Eq. 2nd correctness: C2 = [C1 = 1 and (OOM_jde2 = 0 or OOM_jd1 = 1)]."""
    return int(c1 == 1 and ((oom2 is not None and not oom2) or bool(oom1)))


def memory_saving(c1: int, oom1: bool, oom2: Optional[bool], est: int, m_max: int) -> int:
    """Eq. memory-savings (piecewise, in bytes)."""
    if c1 == 1 and oom2 is not None and not oom2:
        return int(m_max) - int(est)
    if c1 == 1 and oom1:
        return int(m_max)
    return -int(m_max)


def median(xs: List[float]) -> float:
    """Median; an even count takes the mean of the central pair (SPEC D1)."""
    if not xs:
        raise MetricsError("no data")
    s = sorted(xs)
    n = len(s)
    if n % 2:
        return s[n // 2]
    return (s[n // 2 - 1] + s[n // 2]) / 2.0


def check_gating(r: Dict) -> None:
    c1 = correctness1(r["oom_pred"], r["oom1"])
    if r["oom2"] is not None and not (c1 == 1 and not r["oom1"]):
        raise MetricsError("round-2 fields on a run that round 2 excludes (P:385)")


def evaluate(runs: List[Dict]) -> Dict:
    """All metrics over N runs: MRE, PEF (rounds 1 and 2), MCP, and the sums."""
    n = len(runs)
    if n == 0:
        raise MetricsError("no runs")
    errs, c1s, c2s, saves = [], 0, 0, 0
    for r in runs:
        check_gating(r)
        c1 = correctness1(r["oom_pred"], r["oom1"])
        c2 = correctness2(c1, r["oom2"], r["oom1"])
        c1s += c1
        c2s += c2
        saves += memory_saving(c1, r["oom1"], r["oom2"], r["est"], r["m_max"])
        if not r["oom1"]:                                     # OOM_jd1 = 0
            if r["oom2"] is not None and not r["oom2"]:
                errs.append(relative_error(r["est"], r["meas2"]))
            else:
                errs.append(relative_error(r["est"], r["meas1"]))
    return {"n": n, "n_mre": len(errs), "mre": median(errs) if errs else math.nan,
            "pef1": float(n - c1s) / float(n), "pef2": float(n - c2s) / float(n),
            "mcp": float(saves) / float(n), "sum_save": saves, "sum_c1": c1s, "sum_c2": c2s}
