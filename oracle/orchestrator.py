"""ORACLE -- test infrastructure only (see oracle/__init__.py).

The Memory Orchestrator (§3.3;
SPEC.md:151-203 classify_blocks / orchestrate), written out with plain loops:
classify the Analyzer's blocks by the training-loop windows, re-time them
for the analysis iteration, emit the ordered (ts, kind, block) sequence the
Simulator replays.

Input of one trace: blocks in allocation order -- alloc_ts, free_ts (-1 = no
deallocation observed), size, stream -- and per iteration the windows
[start, end] of: iteration, data loading, forward, backward, zero_grad
((-1, -1) if absent), optimizer.step (order of workloads.cpu_profile.WINDOWS).
A window contains ts iff start <= ts <= end (closed, SPEC.md:146 D2).

Classes, first that applies (SPEC D2 priority):
  PARAMETER  no deallocation and allocated before the first iteration (P:241 item 1)
  OPTSTATE   allocated inside an optimizer.step window with a size equal to a
             Parameter's; each Parameter of that size justifies at most two such
             blocks, consumed in allocation order (P:245 item 5; SPEC D3)
  GRADIENT   allocated inside a backward window and not freed before its end
             (P:244 item 4; reading Q23: window form of "backward op that persists")
  BATCHDATA  allocated inside a data-loading window (P:242 item 2)
  ACTIVATION allocated inside a forward or backward window (P:243 item 3)
  OTHER      otherwise
Re-timing for the analysis iteration a = 1 (the second, SPEC D1), window
W = [Ws, We) (reading Q24):
  * a block allocated at or after We, or no longer alive at Ws, is left out;
    a BatchData block's free is first clamped to its iteration's end;
  * allocated before Ws and alive: allocation moves to Ws (carryover);
    Parameter / OptState never free; a Gradient frees at the end of W's
    zero_grad window, at We if W has none (SPEC D5); others keep a
    free before We, else free at We;
  * allocated inside W: allocation kept; Parameter / OptState keep a free
    before We, else none; BatchData frees at min(free, We); a Gradient
    frees at We (its zero_grad is the next iteration's); others keep a free
    before We, else free at We;
  * a moved free never precedes or ties its allocation: F' = max(F', A' + 1).
Output order: (ts, Free before Alloc, block index) (D4).

Parity status: pinned (tests/test_oracle_orchestrator.py: SPEC.md:170-182
worked examples, SPEC.md:183-187 properties, and the generator's ground-truth
kinds for parameters, optimizer state, gradients and batch data).
"""
from __future__ import annotations

from collections import Counter
from typing import Dict, List, Tuple

import numpy as np

PARAMETER, OPTSTATE, GRADIENT, BATCHDATA, ACTIVATION, OTHER = range(6)
CLASS_NAMES = ["Parameter", "OptimizerState", "Gradient", "BatchData", "Activation", "Other"]
IT, DATA, FW, BW, ZG, OPT = range(6)
FREE, ALLOC = 0, 1


class OrchestratorError(ValueError):
    pass


def _inside(ts: int, w) -> bool:
    return w[0] >= 0 and w[0] <= ts <= w[1]


def classify(alloc_ts, free_ts, size, win) -> List[int]:
    n = len(alloc_ts)
    first = int(win[0][IT][0])
    cls = [OTHER] * n
    quota: Counter = Counter()
    for i in range(n):
        if free_ts[i] == -1 and alloc_ts[i] < first:
            cls[i] = PARAMETER
            quota[int(size[i])] += 2
    for i in range(n):
        if cls[i] == PARAMETER:
            continue
        a = int(alloc_ts[i])
        if any(_inside(a, w[OPT]) for w in win) and quota[int(size[i])] > 0:
            quota[int(size[i])] -= 1
            cls[i] = OPTSTATE
        elif any(_inside(a, w[BW]) and (free_ts[i] == -1 or free_ts[i] > w[BW][1]) for w in win):
            cls[i] = GRADIENT
        elif any(_inside(a, w[DATA]) for w in win):
            cls[i] = BATCHDATA
        elif any(_inside(a, w[FW]) or _inside(a, w[BW]) for w in win):
            cls[i] = ACTIVATION
    return cls


def _iter_end(ts: int, win) -> int:
    for w in win:
        if w[IT][0] <= ts <= w[IT][1]:
            return int(w[IT][1])
    return -1


def orchestrate(alloc_ts, free_ts, size, win, a: int = 1) -> Tuple[List[int], List[Tuple[int, int, int]]]:
    """Returns (class per block, sorted events (ts, kind, block index))."""
    if len(win) < a + 1:
        raise OrchestratorError("fewer than two iterations (SPEC.md:166 pre)")
    cls = classify(alloc_ts, free_ts, size, win)
    Ws, We = int(win[a][IT][0]), int(win[a][IT][1])
    zg_end = int(win[a][ZG][1]) if win[a][ZG][0] >= 0 else None
    ev = []
    for i in range(len(alloc_ts)):
        c, A, F = cls[i], int(alloc_ts[i]), int(free_ts[i])
        if A >= We:
            continue
        if c == BATCHDATA:
            e = _iter_end(A, win)
            if e >= 0 and (F == -1 or F > e):
                F = e
        if A < Ws:
            if not (F == -1 or F > Ws):
                continue
            A2 = Ws
            if c in (PARAMETER, OPTSTATE):
                F2 = None
            elif c == GRADIENT:
                F2 = zg_end if zg_end is not None else We
            else:
                F2 = F if (F != -1 and F < We) else We
        else:
            A2 = A
            if c in (PARAMETER, OPTSTATE):
                F2 = F if (F != -1 and F < We) else None
            elif c == GRADIENT:
                F2 = We
            else:
                F2 = F if (F != -1 and F < We) else We
        ev.append((A2, ALLOC, i))
        if F2 is not None:
            ev.append((max(F2, A2 + 1), FREE, i))
    ev.sort()
    return cls, ev


def wire(ev, size, stream):
    """The Simulator input of a sorted sequence: bytes +size / -size and
    tag = block index | stream << 28 (ids are labels; the replay does not
    depend on them)."""
    b = np.array([size[i] if k == ALLOC else -size[i] for (_, k, i) in ev], np.int64)
    t = np.array([i | (int(stream[i]) << 28) for (_, _, i) in ev], np.uint32)
    return b, t
