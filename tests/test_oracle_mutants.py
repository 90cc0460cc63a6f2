"""Mutation check of the oracle's pins.

Each mutant is a plausible one-token mistake in oracle/xmo.c (a dropped term,
a wrong comparison, a swapped operand, a missing step). The test compiles the
mutant to a temporary library and requires that the pins -- the cited hand
goldens plus the gap-model brute force on a small fuzz slice -- reject it.
This is evidence that the pins are strong enough to pin the oracle.
"""
import ctypes
import sys
import os
import subprocess
import tempfile

import numpy as np
import pytest

import bruteforce
import oracle
from workloads import fuzz, hand

SRC = os.path.join(os.path.dirname(oracle.__file__), "xmo.c")

MUTANTS = [
    ("round: drop ceil", "if (q * c->min_block < request) q += 1;", ""),
    ("pool: < instead of <=", "return s <= c->small_size;", "return s < c->small_size;"),
    ("segment: small buffer for large", "if (s < c->min_large_alloc) return c->large_buffer;",
     "if (s < c->min_large_alloc) return c->small_buffer;"),
    ("segment: <= min_large", "if (s < c->min_large_alloc)", "if (s <= c->min_large_alloc)"),
    ("split: small >", "if (small_pool) return remaining >= c->min_block;",
     "if (small_pool) return remaining > c->min_block;"),
    ("split: large never", "if (c->large_split_strict) return remaining > c->small_size;",
     "if (c->large_split_strict) return 0;"),
    ("best fit: ignore stream", "B->small != small || B->stream != stream || B->size < s",
     "B->small != small || B->size < s"),
    ("best fit: worst fit", "B->size < S.blk[best].size ||", "B->size > S.blk[best].size ||"),
    ("best fit: tie by high addr", "B->addr < S.blk[best].addr", "B->addr > S.blk[best].addr"),
    ("capacity: >=", "if (S.reserved + a > cc.capacity) {           /* device refuses",
     "if (S.reserved + a >= cc.capacity) {           /* device refuses"),
    ("no reclamation", "release_cached(&S, out);                /* reclaim",
     "/* release_cached */;                /* reclaim"),
    ("no merge prev", "if (p >= 0 && !S.blk[p].allocated) {", "if (0) {"),
    ("no merge next", "if (q >= 0 && !S.blk[q].allocated) {", "if (0) {"),
    ("split remainder at low end", "R->addr = B->addr + s;", "R->addr = B->addr;"),
    ("reserved not raised", "S.reserved += a;\n", "\n"),
    ("alloc_blk counts request", "S.alloc_blk += S.blk[b].size;", "S.alloc_blk += s;"),
    ("peak idx last", "if (S.reserved > out[F_PEAK_RES])", "if (S.reserved >= out[F_PEAK_RES])"),
    ("release partial segments", "if (b->prev < 0 && b->next < 0) {", "if (b->prev < 0 || b->next < 0) {"),
]


def _build(src_text, d):
    os.makedirs(d, exist_ok=True)
    c = os.path.join(d, "m.c")
    so = os.path.join(d, "m.so")
    with open(c, "w") as f:
        f.write(src_text)
    subprocess.check_call(["gcc", "-O1", "-std=c99", "-shared", "-fPIC", "-w", "-o", so, c])
    L = ctypes.CDLL(so)
    P = ctypes.c_void_p
    L.xmo_simulate.argtypes = [P, P, ctypes.c_int64, ctypes.POINTER(oracle._Cfg), ctypes.c_uint64,
                               P, P, ctypes.c_int]
    return L


def _run(L, by, tg, cap, cfg=None):
    by = np.ascontiguousarray(by, np.int64)
    tg = np.ascontiguousarray(tg, np.uint32)
    out = np.zeros(oracle.NF, np.uint64)
    cv = np.zeros((len(by), 3), np.uint64)
    c = (cfg or oracle.Config()).c()
    rc = L.xmo_simulate(by.ctypes.data_as(P := ctypes.c_void_p), tg.ctypes.data_as(P), len(by),
                        ctypes.byref(c), cap, out.ctypes.data_as(P), cv.ctypes.data_as(P), 0)
    return rc, dict(zip(oracle.FIELDS, map(int, out))), cv


def _pins_reject(L, golden):
    tr = hand.all_named()
    for name, g in golden.items():
        b = tr[name]
        rc, r, _ = _run(L, b.bytes, b.tag, int(b.capacity[0]))
        if rc or any(r[k] != v for k, v in g["expect"].items()):
            return f"golden {name}"
    for corpus in (fuzz.spec1_corpus(120, 400, salt=21), fuzz.capacity_corpus(60, 300, salt=22),
                   fuzz.small_size_corpus(40, 300, salt=23)):
        for t in range(corpus.n_traces):
            by, tg = corpus.trace(t)
            cap = int(corpus.capacity[t])
            rc, r, cv = _run(L, by, tg, cap)
            b, bc = bruteforce.simulate(by, tg, cap)
            if rc or any(r[k] != v for k, v in b.items()):
                return f"bruteforce trace {t}"
            n = b["events_done"]
            if cv[:n].tolist() != [list(x) for x in bc[:n]]:
                return f"bruteforce curve {t}"
    return None


def test_unmutated_passes(golden):
    with tempfile.TemporaryDirectory() as d:
        assert _pins_reject(_build(open(SRC).read(), d), golden) is None


@pytest.mark.parametrize("name,old,new", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_mutant_rejected(name, old, new, golden):
    src = open(SRC).read()
    assert src.count(old) >= 1, f"mutation site missing: {name}"
    with tempfile.TemporaryDirectory() as d:
        L = _build(src.replace(old, new, 1), d)
        assert _pins_reject(L, golden) is not None, f"pins did not catch mutant: {name}"


# ---- NEXT-4 variants (tests/test_oracle_variants.py pins) ----------------------
VARIANT_MUTANTS = [
    ("roundup: interval one power too high", "while (p2 <= request / 2) p2 *= 2;",
     "while (p2 <= request) p2 *= 2;"),
    ("roundup: step 2^k/(2N)", "uint64_t step = p2 / div;", "uint64_t step = p2 / div / 2;"),
    ("roundup: threshold min_block*N/4", "if (div && request > c->min_block * div) {",
     "if (div && request > c->min_block * div / 4) {"),
    ("roundup: floor", "if (k * step < request) k += 1;", ""),
    ("D3: smallest first", "if (best < 0 || b->size > S->blk[S->fr[best]].size ||",
     "if (best < 0 || b->size < S->blk[S->fr[best]].size ||"),
    ("D3: partial segments", "if (b->prev >= 0 || b->next >= 0) continue;",
     "if (b->prev >= 0 && b->next >= 0) continue;"),
    ("D3: release all", "      if (cc.reclaim_policy == 1)", "      if (0)"),
]


def _variant_pins_reject(L):
    from workloads import hand as H
    b = H.h8()
    by, tg = b.trace(0)
    rc, r, _ = _run(L, by, tg, 32 << 20, oracle.Config(reclaim_policy=1))
    if rc or (r["n_seg_release"], r["final_reserved"]) != (1, 14 << 20):
        return "H8"
    for div, corpus in ((4, fuzz.spec1_corpus(60, 300, salt=64)),
                        (2, fuzz.small_size_corpus(30, 300, salt=72)),
                        (0, fuzz.capacity_corpus(60, 300, salt=81))):
        cfg = oracle.Config(roundup_power2_divisions=div, reclaim_policy=int(div == 0))
        for t in range(corpus.n_traces):
            by, tg = corpus.trace(t)
            cap = int(corpus.capacity[t])
            rc, r, cv = _run(L, by, tg, cap, cfg)
            bb, bc = bruteforce.simulate(by, tg, cap, div=div, reclaim=int(div == 0))
            if rc or any(r[k] != v for k, v in bb.items()):
                return f"bruteforce div={div} trace {t}"
    return None


@pytest.mark.parametrize("name,old,new", VARIANT_MUTANTS, ids=[m[0] for m in VARIANT_MUTANTS])
def test_variant_mutant_rejected(name, old, new):
    src = open(SRC).read()
    assert src.count(old) >= 1, f"mutation site missing: {name}"
    with tempfile.TemporaryDirectory() as d:
        assert _variant_pins_reject(_build(src, d)) is None
        L = _build(src.replace(old, new, 1), d + "/m")
        assert _variant_pins_reject(L) is not None, f"pins did not catch mutant: {name}"


# ---- torch knobs max_split_size / garbage_collection_threshold (Q26, Q27) -------
KNOB_MUTANTS = [
    ("msplit: small request takes an oversize block",
     "if (s < cc.max_split_size && bs >= cc.max_split_size) best = -1;", "if (0) best = -1;"),
    ("msplit: no non-split rounding bound",
     "else if (s >= cc.max_split_size && bs >= s + cc.max_non_split_rounding) best = -1;", ""),
    ("msplit: oversize requests split", "&& (small || s < cc.max_split_size)", "&& (1)"),
    ("release_available: largest fitting block",
     "if (best < 0 || B->size < S->blk[S->fr[best]].size ||",
     "if (best < 0 || B->size > S->blk[S->fr[best]].size ||"),
    ("release_available: a failed walk still retries", "return released >= key ? 1 : 0;", "return 1;"),
    ("release_available: never", "int e = release_available(&S, &cc, s, small, stream, out);",
     "int e = 0;"),
    ("GC: strictly older than the mean", "(double)age >= age_threshold", "(double)age > age_threshold"),
    ("GC: small pool counted", "if (B->small || B->prev >= 0 || B->next >= 0) continue;",
     "if (B->prev >= 0 || B->next >= 0) continue;"),
    ("GC: one pass only", "while (reclaimed < target && freed && freeable > 0) {",
     "while (reclaimed < target && freed && freeable > 0 && !reclaimed) {"),
    ("GC: bar from reserved", "(uint64_t)(c->gc_threshold * (double)c->capacity)",
     "(uint64_t)(c->gc_threshold * (double)S->reserved)"),
    ("GC: age never reset", "  S->blk[b].gc_base = S->searches[S->blk[b].small];\n", ""),
]


def _knob_pins_reject(L):
    import test_oracle_variants as V
    M = 1 << 20
    hand_cases = [  # (events, capacity, msplit, gc, expected fields) from the H9-H12 docstrings
        (lambda t: t.alloc(0, 100 * M).free(0).alloc(1, 90 * M).free(1).alloc(2, 30 * M)
         .alloc(3, 70 * M), oracle.UNLIMITED, 64 * M, 0.0, {"peak_reserved": 200 * M}),
        (lambda t: t.alloc(0, 100 * M).alloc(1, 30 * M).alloc(2, M).free(0).free(1).free(2)
         .alloc(3, 70 * M), 180 * M, 64 * M, 0.0, {"n_seg_release": 1, "final_reserved": 102 * M}),
        (lambda t: t.alloc(0, 66 * M).alloc(1, 70 * M).alloc(2, 30 * M).free(0).free(1).free(2)
         .alloc(3, 120 * M), 200 * M, 64 * M, 0.0, {"n_seg_release": 2, "final_reserved": 150 * M}),
        (lambda t: t.alloc(0, 66 * M).alloc(1, 70 * M).alloc(2, 30 * M).free(0).free(1).free(2)
         .alloc(3, 150 * M), 200 * M, 64 * M, 0.0, {"n_seg_release": 3}),
        (lambda t: t.alloc(0, 200 * M).alloc(1, 150 * M).alloc(2, 120 * M).alloc(3, 60 * M).free(0)
         .free(2).alloc(4, 110 * M).free(4).alloc(5, 100 * M).free(5).alloc(6, 300 * M),
         1000 * M, None, 0.5, {"peak_reserved": 630 * M, "n_seg_release": 1}),
    ]
    for k, (ev, cap, ms, gc, exp) in enumerate(hand_cases):
        by, tg = V._one(ev, cap)
        cfg = oracle.Config(gc_threshold=gc, **({"max_split_size": ms} if ms else {}))
        rc, r, _ = _run(L, by, tg, cap, cfg)
        if rc or any(r[f] != v for f, v in exp.items()):
            return f"hand H{9 + k}"
    for ms, gc, corpus in ((24 * M, 0.0, fuzz.spec1_corpus(50, 300, salt=94)),
                           (24 * M, 0.0, fuzz.capacity_corpus(60, 300, salt=95)),
                           (None, 0.5, fuzz.capacity_corpus(60, 300, salt=96)),
                           (None, 0.3, fuzz.capacity_corpus(60, 300, salt=97))):
        cfg = oracle.Config(gc_threshold=gc, **({"max_split_size": ms} if ms else {}))
        for t in range(corpus.n_traces):
            by, tg = corpus.trace(t)
            cap = int(corpus.capacity[t])
            rc, r, _ = _run(L, by, tg, cap, cfg)
            bb, _ = bruteforce.simulate(by, tg, cap, msplit=ms, gc=gc)
            if rc or any(r[k] != v for k, v in bb.items()):
                return f"bruteforce msplit={ms} gc={gc} trace {t}"
    return None


@pytest.mark.parametrize("name,old,new", KNOB_MUTANTS, ids=[m[0] for m in KNOB_MUTANTS])
def test_knob_mutant_rejected(name, old, new):
    src = open(SRC).read()
    assert src.count(old) >= 1, f"mutation site missing: {name}"
    with tempfile.TemporaryDirectory() as d:
        assert _knob_pins_reject(_build(src, d)) is None
        L = _build(src.replace(old, new, 1), d + "/m")
        assert _knob_pins_reject(L) is not None, f"pins did not catch mutant: {name}"


# ---- NEXT-3 lifecycle oracle (oracle/lifecycle.c) -------------------------------
LC_SRC = os.path.join(os.path.dirname(oracle.__file__), "lifecycle.c")
LC_MUTANTS = [
    ("pop empties the address", "s->top = below[b];", "s->top = -1;"),
    ("mismatch sign", "if (bytes[b] != -bytes[i])", "if (bytes[b] != bytes[i])"),
    ("orphan closes nothing but counts", "tallies[1] += 1;", ""),
    ("push keeps old top", "below[i] = s->top;\n      s->top = i;", "below[i] = -1;\n      s->top = i;"),
    ("persistent count", "tallies[3] = open;", "tallies[3] = tallies[0] - open;"),
]


def _lc_build(src_text, d):
    os.makedirs(d, exist_ok=True)
    c = os.path.join(d, "lc.c")
    so = os.path.join(d, "lc.so")
    with open(c, "w") as f:
        f.write(src_text)
    subprocess.check_call(["gcc", "-O1", "-std=c99", "-shared", "-fPIC", "-w", "-o", so, c])
    L = ctypes.CDLL(so)
    P = ctypes.c_void_p
    L.xmo_reconstruct.argtypes = [P, P, ctypes.c_int64, P, P, P]
    return L


def _lc_pins_reject(L):
    import test_oracle_lifecycle as TL
    from workloads import instants
    P = ctypes.c_void_p

    def rec(a, by):
        a = np.ascontiguousarray(a, np.uint64)
        by = np.ascontiguousarray(by, np.int64)
        p = np.zeros(len(by), np.int64)
        m = np.zeros(len(by), np.uint8)
        t = np.zeros(6, np.uint64)
        rc = L.xmo_reconstruct(a.ctypes.data_as(P), by.ctypes.data_as(P), len(by),
                               p.ctypes.data_as(P), m.ctypes.data_as(P), t.ctypes.data_as(P))
        return rc, p, m, t
    # SPEC examples + LIFO / mismatch cases
    cases = [([0xA, 0xA], [1024, -1024], [1, 0], [1, 0, 0, 0]), ([0xB], [-512], [-1], [0, 1, 0, 0]),
             ([5, 5, 5, 5], [100, 200, -200, -100], [3, 2, 1, 0], [2, 0, 0, 0]),
             ([5, 5], [100, -96], [1, 0], [1, 0, 1, 0]), ([7, 7, 7], [8, -8, 16], [1, 0, -1], [2, 0, 0, 1])]
    for a, by, part, tal in cases:
        rc, p, m, t = rec(a, by)
        if rc or p.tolist() != part or t[:4].tolist() != tal:
            return f"case {a}"
    b = fuzz.spec1_corpus(20, 300, salt=31)
    ins = instants.from_batch(b, salt=1, p_orphan=0.02, p_mismatch=0.02, p_lost=0.03)
    for t in range(ins.n_traces):
        a, by, st = ins.trace(t)
        rc, p, m, tal = rec(a, by)
        if rc or p.tolist() != TL.brute(a.tolist(), by.tolist()):
            return f"brute trace {t}"
    return None


@pytest.mark.parametrize("name,old,new", LC_MUTANTS, ids=[m[0] for m in LC_MUTANTS])
def test_lifecycle_mutant_rejected(name, old, new):
    src = open(LC_SRC).read()
    assert src.count(old) >= 1, f"mutation site missing: {name}"
    with tempfile.TemporaryDirectory() as d:
        assert _lc_pins_reject(_lc_build(src, d)) is None
        assert _lc_pins_reject(_lc_build(src.replace(old, new, 1), d + "/m")) is not None, name


# ---- NEXT-2 orchestrator and NEXT-4 metrics oracles (Python) ---------------------
PY_MUTANTS = [
    ("orchestrator", "quota 1 per parameter", "quota[int(size[i])] += 2", "quota[int(size[i])] += 1"),
    ("orchestrator", "gradient needs no survival", "(free_ts[i] == -1 or free_ts[i] > w[BW][1])", "True"),
    ("orchestrator", "open window bounds", "return w[0] >= 0 and w[0] <= ts <= w[1]", "return w[0] >= 0 and w[0] < ts < w[1]"),
    ("orchestrator", "carried gradient at We", "F2 = zg_end if zg_end is not None else We", "F2 = We"),
    ("orchestrator", "batch data not clamped", "if e >= 0 and (F == -1 or F > e):", "if False:"),
    ("orchestrator", "Alloc before Free on ties", "FREE, ALLOC = 0, 1", "FREE, ALLOC = 1, 0"),
    ("metrics", "median upper", "return (s[n // 2 - 1] + s[n // 2]) / 2.0", "return s[n // 2]"),
    ("metrics", "C2 without OOM_jd1", "return int(c1 == 1 and ((oom2 is not None and not oom2) or bool(oom1)))",
     "return int(c1 == 1 and (oom2 is not None and not oom2))"),
    ("metrics", "saving sign", "    return -int(m_max)", "    return int(m_max)"),
    ("metrics", "MRE uses round 1 always", 'errs.append(relative_error(r["est"], r["meas2"]))',
     'errs.append(relative_error(r["est"], r["meas1"]))'),
]


@pytest.mark.parametrize("mod,name,old,new", PY_MUTANTS, ids=[m[1] for m in PY_MUTANTS])
def test_python_oracle_mutant_rejected(mod, name, old, new, monkeypatch):
    import importlib
    import types
    path = os.path.join(os.path.dirname(oracle.__file__), f"{mod}.py")
    src = open(path).read()
    assert src.count(old) >= 1, f"mutation site missing: {name}"
    m = types.ModuleType(f"oracle.{mod}")
    exec(compile(src.replace(old, new, 1), path, "exec"), m.__dict__)
    monkeypatch.setitem(sys.modules, f"oracle.{mod}", m)
    monkeypatch.setattr(oracle, mod, m, raising=False)
    test_mod = importlib.import_module(f"test_oracle_{'orchestrator' if mod == 'orchestrator' else 'metrics'}")
    importlib.reload(test_mod)
    failed = False
    for k, fn in vars(test_mod).items():
        if not k.startswith("test_") or not callable(fn):
            continue
        try:
            args = []
            import inspect
            params = inspect.signature(fn).parameters
            if params:
                # parametrized examples: run their table
                marks = getattr(fn, "pytestmark", [])
                for mk in marks:
                    if mk.name == "parametrize":
                        for vals in mk.args[1]:
                            fn(*vals)
                continue
            fn()
        except Exception:
            failed = True
            break
    monkeypatch.undo()                 # the real oracle module back, then rebind
    importlib.reload(test_mod)
    assert failed, f"pins did not catch mutant: {name}"
