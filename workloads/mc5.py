"""Config 5 (BASELINE configs[4]): Monte Carlo traces at paper scale (1M), built
from ~200 dense templates by a COUNTER-BASED recipe that the GPU expander K4
(paper_2510_21048_b200/csrc/expand.cu, xm_expand_templates) implements too, so
a 1M-trace batch is generated on the device while any single trace can be
rebuilt here, on the host, for the oracle (DESIGN.md §4 "Config 5").

Input generation only (no allocator arithmetic; see the package docstring).

Recipe for global trace index i (salt 7):
  sigma_i  = splitmix64(0x784D656D ^ i ^ salt << 32)              (rng.trace_seed)
  draw k   = splitmix64(sigma_i ^ k << 56), k = 1..5 -> model (22 RQ1-RQ4 models,
             PAPER.md:337-371), optimizer, batch size, zero_grad placement
             (PAPER.md:105-111), capacity 12 / 8 GiB (RTX 3060 / 4060)
  template = models.template(model, opt, zero_grad, img=32, seq=512), with block
             ids renumbered densely (a freed id is reused LIFO by the next alloc)
  swaps    = CPU-timing jitter (PAPER.md:248 footnote): c(j) = splitmix64(sigma_i
             + j + 1) < 0.02 * 2^64 marks a candidate swap of positions (j, j+1),
             j <= n-2; it is applied iff c(j) and not c(j-1) and the two events
             carry different ids. Event j then takes its content from j+1 (swap
             at j), j-1 (swap at j-1) or j.
  event    = bytes (fixed + per_sample * b) * sign, tag = dense id | stream << 28
"""
from __future__ import annotations

from functools import lru_cache
from typing import List, Tuple

import numpy as np

from . import models as M
from .rng import SEED_BASE
from .trace import Batch

GiB = 1 << 30
SALT = 7
SWAP_P = 0.02
SWAP_THRESHOLD = int(SWAP_P * 2.0 ** 64)           # c(j) iff hash < this
IMG, SEQ = 32, 512
MODELS = M.CNNS_PAPER + M.TRANSFORMERS + M.SMALL_LLMS          # 22 models
CNN_OPTS = ["sgd", "adam", "adamw", "rmsprop", "adagrad"]
TR_OPTS = ["sgd", "adafactor", "adam", "adamw"]
ZG = ["pos0", "pos1"]
CAPS = [12 * GiB, 8 * GiB]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _opts(name):
    return CNN_OPTS if name in M.CNNS_PAPER else TR_OPTS


def _batches(name):
    if name in M.CNNS_PAPER:
        return list(range(200, 701, 100))
    if name in M.SMALL_LLMS:
        return list(range(1, 9))
    return list(range(5, 56, 5))


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 (wrapping uint64 arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def seeds(idx: np.ndarray, salt: int = SALT) -> np.ndarray:
    idx = np.asarray(idx, np.uint64)
    return splitmix64_np(np.uint64(SEED_BASE) ^ idx ^ np.uint64((salt << 32) & 0xFFFFFFFFFFFFFFFF))


# ---- templates ---------------------------------------------------------------
TEMPLATES: List[Tuple[str, str, str]] = [(m, o, z) for m in MODELS for o in _opts(m) for z in ZG]
_TPL_INDEX = {k: i for i, k in enumerate(TEMPLATES)}


def dense_ids(bid: np.ndarray, sign: np.ndarray) -> Tuple[np.ndarray, int]:
    """Renumber block ids densely: an alloc takes the most recently freed id
    (LIFO) or a fresh one. Returns (ids, id space)."""
    out = np.empty(len(bid), np.uint32)
    live = {}
    free: List[int] = []
    nxt = 0
    for j in range(len(bid)):
        b = int(bid[j])
        if sign[j] > 0:
            if free:
                d = free.pop()
            else:
                d = nxt
                nxt += 1
            live[b] = d
            out[j] = d
        else:
            d = live.pop(b)
            out[j] = d
            free.append(d)
    return out, nxt


@lru_cache(maxsize=None)
def template(k: int):
    """Template k: (fixed int64 signed, per int64 signed, tag uint32, id space)."""
    name, opt, zg = TEMPLATES[k]
    sign, fixed, per, bid, stream = M.template(name, opt, zg, img=IMG, seq=SEQ)
    ids, nids = dense_ids(bid, sign)
    tag = (ids | (stream.astype(np.uint32) << np.uint32(28))).astype(np.uint32)
    return (fixed * sign).astype(np.int64), (per * sign).astype(np.int64), tag, nids


@lru_cache(maxsize=1)
def template_pool():
    """All templates concatenated: (fixed, per, tag, tpl_off[n_tpl+1], n_ids[n_tpl])."""
    parts = [template(k) for k in range(len(TEMPLATES))]
    off = np.zeros(len(parts) + 1, np.int64)
    off[1:] = np.cumsum([len(p[0]) for p in parts])
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]),
            np.concatenate([p[2] for p in parts]), off,
            np.array([p[3] for p in parts], np.uint32))


# ---- descriptors ---------------------------------------------------------------
def _tables():
    tpl_of = np.zeros((len(MODELS), 5, 2), np.int32)
    nb = np.zeros(len(MODELS), np.int64)
    nopt = np.zeros(len(MODELS), np.int64)
    btab = np.zeros((len(MODELS), 11), np.int64)
    for mi, m in enumerate(MODELS):
        nopt[mi] = len(_opts(m))
        bs = _batches(m)
        nb[mi] = len(bs)
        btab[mi, :len(bs)] = bs
        for oi, o in enumerate(_opts(m)):
            for zi, z in enumerate(ZG):
                tpl_of[mi, oi, zi] = _TPL_INDEX[(m, o, z)]
    return tpl_of, nb, nopt, btab


def describe(idx, salt: int = SALT):
    """Per-trace descriptors of global indices idx: dict of arrays
    tpl (template index), b (batch size), capacity, seed."""
    idx = np.asarray(idx, np.int64)
    sig = seeds(idx, salt)
    r = [splitmix64_np(sig ^ np.uint64(k << 56)) for k in range(1, 6)]
    tpl_of, nb, nopt, btab = _tables()
    mi = (r[0] % np.uint64(len(MODELS))).astype(np.int64)
    oi = (r[1] % nopt[mi].astype(np.uint64)).astype(np.int64)
    bi = (r[2] % nb[mi].astype(np.uint64)).astype(np.int64)
    zi = (r[3] & np.uint64(1)).astype(np.int64)
    ci = (r[4] & np.uint64(1)).astype(np.int64)
    return {"tpl": tpl_of[mi, oi, zi].astype(np.uint32), "b": btab[mi, bi].astype(np.uint32),
            "capacity": np.array(CAPS, np.uint64)[ci], "seed": sig}


def lengths(desc) -> np.ndarray:
    off = template_pool()[3]
    return np.diff(off)[desc["tpl"]]


# ---- host instantiation (for the oracle / parity samples) ----------------------
def swap_source(n: int, seed: np.uint64) -> np.ndarray:
    """c[j]: position j starts a candidate swap (j, j+1) (before the adjacency and
    same-id filters)."""
    j = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64_np(np.uint64(seed) + j + np.uint64(1))
    c = h < np.uint64(SWAP_THRESHOLD)
    if n > 0:
        c[n - 1] = False                      # no pair (n-1, n)
    return c


def instantiate(k: int, b: int, seed) -> Tuple[np.ndarray, np.ndarray]:
    fixed, per, tag, _ = template(k)
    n = len(fixed)
    c = swap_source(n, np.uint64(seed))
    keep = c.copy()
    keep[1:] &= ~c[:-1]
    ids = tag & np.uint32(0x0FFFFFFF)
    keep[:-1] &= ids[:-1] != ids[1:]            # same block id -> no swap
    keep[n - 1:] = False
    src = np.arange(n)
    ks = np.flatnonzero(keep)
    src[ks] = ks + 1
    src[ks + 1] = ks
    by = fixed[src] + per[src] * np.int64(b)
    return by.astype(np.int64), tag[src].astype(np.uint32)


def batch(idx, salt: int = SALT) -> Batch:
    """Host-built config-5 traces with global indices idx (caller order)."""
    idx = np.asarray(idx, np.int64)
    d = describe(idx, salt)
    items = [instantiate(int(d["tpl"][t]), int(d["b"][t]), d["seed"][t]) for t in range(len(idx))]
    off = np.zeros(len(idx) + 1, np.int64)
    off[1:] = np.cumsum([len(it[0]) for it in items])
    names = [f"mc5:{int(i)}:" + "/".join(TEMPLATES[int(d['tpl'][t])]) + f"/b{int(d['b'][t])}"
             for t, i in enumerate(idx)]
    return Batch(np.concatenate([it[0] for it in items]) if items else np.zeros(0, np.int64),
                 np.concatenate([it[1] for it in items]) if items else np.zeros(0, np.uint32),
                 off, d["capacity"].astype(np.uint64), names)


# ---- the same recipe in C (workloads/mc5gen.c), for full-size host parity ------
_HERE = __import__("os").path.dirname(__import__("os").path.abspath(__file__))
_GEN_SRC = _HERE + "/mc5gen.c"
_GEN_LIB = _HERE + "/libmc5gen.so"
_gen = None


def build_gen(force: bool = False) -> str:
    import os
    import subprocess
    if force or not os.path.exists(_GEN_LIB) or os.path.getmtime(_GEN_LIB) < os.path.getmtime(_GEN_SRC):
        tmp = _GEN_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", "-o", tmp, _GEN_SRC])
        os.replace(tmp, _GEN_LIB)
    return _GEN_LIB


def _genlib():
    global _gen
    if _gen is None:
        import ctypes
        build_gen()
        L = ctypes.CDLL(_GEN_LIB)
        P = ctypes.c_void_p
        L.mc5_instantiate.argtypes = [P, P, P, P, P, P, P, ctypes.c_int64, ctypes.c_uint64, P, P, P]
        L.mc5_instantiate.restype = ctypes.c_int
        _gen = L
    return _gen


def batch_fast(idx, salt: int = SALT) -> Batch:
    """batch(idx) built by the C form of the recipe (byte-identical to batch();
    tests/test_mc5_cpu.py), ~100x faster: the host side of config-5 parity on
    every one of the 1M traces."""
    import ctypes
    idx = np.asarray(idx, np.int64)
    d = describe(idx, salt)
    fixed, per, tag, tpl_off, _ = template_pool()
    n = np.diff(tpl_off)[d["tpl"]]
    off = np.zeros(len(idx) + 1, np.int64)
    off[1:] = np.cumsum(n)
    ob = np.empty(int(off[-1]), np.int64)
    ot = np.empty(int(off[-1]), np.uint32)
    tp = np.ascontiguousarray(d["tpl"], np.uint32)
    bb = np.ascontiguousarray(d["b"], np.uint32)
    sd = np.ascontiguousarray(d["seed"], np.uint64)

    def p(a):
        return a.ctypes.data_as(ctypes.c_void_p)
    rc = _genlib().mc5_instantiate(p(fixed), p(per), p(tag), p(tpl_off), p(tp), p(bb), p(sd),
                                   len(idx), SWAP_THRESHOLD, p(off), p(ob), p(ot))
    if rc:
        raise RuntimeError("mc5_instantiate: span mismatch")
    return Batch(ob, ot, off, d["capacity"].astype(np.uint64), [])
