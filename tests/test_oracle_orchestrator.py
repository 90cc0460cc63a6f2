"""Pins of the orchestrator oracle (oracle/orchestrator.py; SURVEY NEXT-2;
PAPER.md:239-248). No GPU."""
import numpy as np
import pytest

from oracle import orchestrator as O
from workloads import cpu_profile as C


def _win(its):
    """its: list of dicts of window name -> (start, end)."""
    w = np.full((len(its), 6, 2), -1, np.int64)
    for k, d in enumerate(its):
        for name, (s, e) in d.items():
            w[k, C.WINDOWS.index(name)] = (s, e)
    return w


ITS = [dict(iter=(100, 199), data=(100, 105), fw=(106, 140), zg=(141, 145), bw=(146, 170), opt=(171, 199)),
       dict(iter=(200, 299), data=(200, 205), fw=(206, 240), zg=(241, 245), bw=(246, 270), opt=(271, 299)),
       dict(iter=(300, 399), data=(300, 305), fw=(306, 340), zg=(341, 345), bw=(346, 370), opt=(371, 399))]


def test_classify_spec_examples():
    W = _win(ITS)
    a = np.array([10, 180, 120])                # param; in optimizer.step; in forward
    f = np.array([-1, -1, 130])
    s = np.array([4_096_000, 4_096_000, 512])
    cls = O.classify(a, f, s, W)
    assert cls == [O.PARAMETER, O.OPTSTATE, O.ACTIVATION]
    # no matching parameter size -> not optimizer state
    assert O.classify(a, f, np.array([4_096_000, 4_096_004, 512]), W)[1] == O.OTHER


def test_optimizer_state_quota():             # SPEC D3: two per parameter, allocation order
    W = _win(ITS)
    a = np.array([10, 172, 173, 174, 175])
    f = np.array([-1, -1, -1, -1, 176])
    s = np.array([64, 64, 64, 64, 64])
    assert O.classify(a, f, s, W) == [O.PARAMETER, O.OPTSTATE, O.OPTSTATE, O.OTHER, O.OTHER]


def test_orchestrate_spec_examples():
    # windows with the analysis iteration's zero_grad at [180, 185] and end 200
    its = [dict(iter=(50, 99), data=(50, 55), fw=(56, 70), zg=(71, 72), bw=(73, 90), opt=(91, 99)),
           dict(iter=(100, 200), data=(100, 105), fw=(106, 150), zg=(180, 185), bw=(151, 179), opt=(186, 200)),
           dict(iter=(201, 300), data=(201, 205), fw=(206, 250), zg=(251, 252), bw=(253, 280), opt=(281, 300))]
    W = _win(its)
    a = np.array([10, 80, 102])       # param; gradient of iteration 1 (CPU free at 150); batch data
    f = np.array([-1, 150, 230])      # batch freed after the iteration end (200)
    s = np.array([1024, 2048, 4096])
    cls, ev = O.orchestrate(a, f, s, W)
    assert cls == [O.PARAMETER, O.GRADIENT, O.BATCHDATA]
    assert (100, O.ALLOC, 0) in ev and not any(k == O.FREE and i == 0 for (_, k, i) in ev)
    assert (185, O.FREE, 1) in ev                      # gradient free -> zero_grad end
    assert (200, O.FREE, 2) in ev                      # batch data clamped to iteration end


def test_orchestrate_properties():
    p = C.batch([("resnet50", "adam", "pos0", 64, False), ("gpt2", "adamw", "pos1", 5, True),
                 ("mobilenet_v2", "sgd", "pos1", 200, False)])
    for t in range(p.n_traces):
        a, f, s, st, W = p.trace(t)
        cls, ev = O.orchestrate(a, f, s, W)
        assert ev == sorted(ev)                                     # ordering invariant
        Ws, We = W[1][0]
        seen = {}
        for (ts, k, i) in ev:
            assert Ws <= ts <= We
            if k == O.ALLOC:
                assert i not in seen
                seen[i] = ts
            else:
                assert i in seen and ts > seen[i]                   # Free after its Alloc
        for (ts, k, i) in ev:                                       # activations keep times
            if cls[i] == O.ACTIVATION and a[i] >= Ws and k == O.ALLOC:
                assert ts == a[i]
            if cls[i] == O.ACTIVATION and a[i] >= Ws and k == O.FREE and 0 <= f[i] < We:
                assert ts == f[i]
            if cls[i] == O.GRADIENT and k == O.FREE and a[i] < Ws:  # carried-over gradients
                assert ts == (W[1][4][1] if W[1][4][0] >= 0 else We)


def test_classification_matches_generator_truth():
    """The generator knows what each block is; the window rules must recover
    parameters, optimizer state, gradients and batch data exactly."""
    cells = [("resnet50", "adam", "pos0", 64, False), ("gpt2", "adamw", "pos1", 5, True),
             ("vgg16", "rmsprop", "pos0", 200, False), ("t5_small", "adafactor", "pos1", 10, False),
             ("mobilenet_v2", "sgd", "pos1", 300, False)]
    p = C.batch(cells)
    K = C.KINDS
    want = {"param": O.PARAMETER, "state": O.OPTSTATE, "grad": O.GRADIENT, "data": O.BATCHDATA}
    for t in range(p.n_traces):
        a, f, s, st, W = p.trace(t)
        cls = O.classify(a, f, s, W)
        kinds = p.kind[p.boff[t]:p.boff[t + 1]]
        psizes = {int(s[i]) for i, k in enumerate(kinds) if K[k] == "param"}
        for i, k in enumerate(kinds):
            if K[k] == "state" and (int(s[i]) not in psizes or "adafactor" in p.names[t]):
                # factored states (Adafactor row/column vectors) do not match the
                # parameter sizes one to one: the size heuristic and its
                # quota (SPEC D3) cannot always see them
                assert cls[i] in (O.OPTSTATE, O.ACTIVATION, O.OTHER), (p.names[t], i, cls[i])
            elif K[k] in want:
                assert cls[i] == want[K[k]], (p.names[t], i, K[k], cls[i])
            elif K[k] == "temp":
                # foreach temporaries of optimizers with one state per parameter
                # fall under SPEC D3's quota of two (the heuristic's known limit)
                assert cls[i] in (O.OPTSTATE, O.ACTIVATION, O.OTHER), (p.names[t], i, cls[i])
            else:
                assert cls[i] in (O.ACTIVATION, O.OTHER), (p.names[t], i, K[k], cls[i])


def test_needs_two_iterations():
    W = _win(ITS[:1])
    with pytest.raises(O.OrchestratorError):
        O.orchestrate(np.array([1]), np.array([-1]), np.array([8]), W)


def test_window_bounds_are_closed():
    """Windows contain their end points (closed bounds, as SPEC.md:146 D2 fixes
    for operator windows): an allocation exactly at a window's start or end
    belongs to it."""
    W = _win(ITS)
    a = np.array([10, 171, 199, 146, 170, 100])
    f = np.array([-1, -1, -1, 180, 185, 150])
    s = np.array([64, 64, 64, 8, 8, 8])
    cls = O.classify(a, f, s, W)
    assert cls == [O.PARAMETER, O.OPTSTATE, O.OPTSTATE, O.GRADIENT, O.GRADIENT, O.BATCHDATA]


def test_previous_batch_does_not_carry_over():
    """P:242 "Batch Data ... lifecycles limited within one training iteration":
    the batch of iteration 1, freed on the CPU only when iteration 2 loads the
    next batch, must not appear in iteration 2's sequence."""
    W = _win(ITS)
    a = np.array([101, 201])          # batch of iteration 1, batch of iteration 2
    f = np.array([202, 302])          # each freed when the next batch loads
    s = np.array([4096, 4096])
    cls, ev = O.orchestrate(a, f, s, W)
    assert cls == [O.BATCHDATA, O.BATCHDATA]
    assert ev == [(201, O.ALLOC, 1), (299, O.FREE, 1)]


def test_free_before_alloc_on_equal_timestamps():
    """SPEC.md:162 / D4: events are ordered by (ts, Free before Alloc, block)."""
    W = _win(ITS)
    a = np.array([210, 230])
    f = np.array([230, 235])
    s = np.array([512, 512])
    cls, ev = O.orchestrate(a, f, s, W)
    assert ev == [(210, O.ALLOC, 0), (230, O.FREE, 0), (230, O.ALLOC, 1), (235, O.FREE, 1)]
