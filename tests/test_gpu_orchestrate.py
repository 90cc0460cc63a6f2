"""NEXT-2 memory orchestrator on the GPU (xm_orchestrate, K6) vs the oracle
(oracle/orchestrator.py): classes of every block, the re-timed sorted
sequence of every trace, the per-trace records, the wire form (bytes equal,
ids valid) and its replay (K2) vs the oracle's replay, bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle
import paper_2510_21048_b200 as xm
from gpu_util import assert_parity
from oracle import orchestrator as O
from workloads import cpu_profile as C
from workloads.trace import Batch


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _synthetic(n_blocks, seed, iters=3):
    """Hand-rolled profile: many blocks across windows, random lifetimes."""
    rng = np.random.default_rng(seed)
    win = np.full((iters, 6, 2), -1, np.int64)
    for k in range(iters):
        s = 1000 + k * 100000
        win[k] = [(s, s + 99990), (s, s + 99), (s + 100, s + 40000), (s + 50000, s + 80000),
                  (s + 40001, s + 49999) if k % 2 else (-1, -1), (s + 80001, s + 99990)]
    a = np.sort(rng.integers(0, 1000 + iters * 100000, n_blocks))
    life = rng.integers(1, 60000, n_blocks)
    f = np.where(rng.random(n_blocks) < 0.1, -1, a + life)
    size = rng.choice([512, 4096, 65536, 1 << 20, 3 << 20], n_blocks)
    size[a < 1000] = rng.choice([4096, 65536], int((a < 1000).sum()))
    return a.astype(np.int64), f.astype(np.int64), size.astype(np.int64), \
        rng.integers(0, 3, n_blocks).astype(np.uint8), win


def _profiles():
    cells = [("resnet50", "adam", "pos0", 64, False), ("gpt2", "adamw", "pos1", 5, True),
             ("vgg16", "rmsprop", "pos0", 200, False), ("t5_small", "adafactor", "pos1", 10, False),
             ("mobilenet_v2", "sgd", "pos1", 300, False), ("bert_base", "adamw", "pos0", 15, True)]
    p = C.batch(cells)
    # append synthetic traces: a big one (9000 blocks: global-memory sort), a
    # one-iteration one (status), an empty one
    extra = [_synthetic(9000, 1), _synthetic(300, 2, iters=1), _synthetic(0, 3)]
    A = [p.alloc_ts] + [e[0] for e in extra]
    F = [p.free_ts] + [e[1] for e in extra]
    S = [p.size] + [e[2] for e in extra]
    ST = [p.stream] + [e[3] for e in extra]
    Wn = [p.win] + [e[4] for e in extra]
    boff = list(p.boff)
    woff = list(p.woff)
    for e in extra:
        boff.append(boff[-1] + len(e[0]))
        woff.append(woff[-1] + len(e[4]))
    return C.Profiles(np.concatenate(A), np.concatenate(F), np.concatenate(S), np.concatenate(ST),
                      np.zeros(boff[-1], np.uint8), np.asarray(boff, np.int64), np.concatenate(Wn),
                      np.asarray(woff, np.int64), p.names + ["synth9000", "synth1it", "empty"])


def test_orchestrate_parity():
    p = _profiles()
    d = xm.DeviceProfiles.from_host(p)
    cls, seq, rec, wb = xm.orchestrate(d)
    cls = cls.cpu().numpy()
    seq = seq.cpu().numpy().view(np.uint64)
    order = wb.order.cpu().numpy().view(np.uint32)
    pos = np.empty(p.n_traces, np.int64)
    pos[order] = np.arange(p.n_traces)
    woff = wb.off.cpu().numpy()
    wbytes = wb.bytes.cpu().numpy()
    wtag = wb.tag.cpu().numpy().view(np.uint32)
    o_wires = []
    for t in range(p.n_traces):
        a, f, s, st, W = p.trace(t)
        b0 = int(p.boff[t])
        if len(W) < 2:
            assert rec["status"][t] == xm_status_few()
            o_wires.append((np.zeros(0, np.int64), np.zeros(0, np.uint32)))
            continue
        ocls, oev = O.orchestrate(a, f, s, W)
        assert rec["status"][t] == 0
        assert (cls[b0:b0 + len(a)] == np.asarray(ocls, np.uint8)).all(), p.names[t]
        assert rec["n_class"][t].tolist() == np.bincount(np.asarray(ocls, np.int64), minlength=6).tolist()
        ws = int(rec["ws"][t])
        assert ws == W[1][0][0] and int(rec["we"][t]) == W[1][0][1]
        n = int(rec["n_events"][t])
        keys = seq[2 * b0:2 * b0 + n]
        gev = [(ws + int(k >> 32), int((k >> 31) & 1), int(k & 0x7FFFFFFF)) for k in keys]
        assert gev == oev, (p.names[t], next(i for i, (x, y) in enumerate(zip(gev, oev)) if x != y))
        ob, ot = O.wire(oev, s, st)
        q = pos[t]
        gb = wbytes[woff[q]:woff[q + 1]]
        gt = wtag[woff[q]:woff[q + 1]]
        assert (gb == ob).all() and ((gt >> 28) == (ot >> 28)).all(), p.names[t]
        live = {}
        for j, (_, k, i) in enumerate(oev):                 # ids: one per open block
            gid = int(gt[j] & 0x0FFFFFFF)
            if k == O.ALLOC:
                assert gid not in live.values()
                live[i] = gid
            else:
                assert live.pop(i) == gid
        o_wires.append((ob, ot))
    # replay of the GPU wire batch == oracle replay of the oracle's sequences
    ok = [t for t in range(p.n_traces) if len(p.trace(t)[4]) >= 2]
    h, _ = xm.peaks(xm.simulate_batch(wb))
    off = np.zeros(len(ok) + 1, np.int64)
    off[1:] = np.cumsum([len(o_wires[t][0]) for t in ok])
    ob = Batch(np.concatenate([o_wires[t][0] for t in ok]), np.concatenate([o_wires[t][1] for t in ok]),
               off, np.full(len(ok), oracle.UNLIMITED, np.uint64))
    assert_parity(ob, h[ok], oracle.simulate_batch(ob))


def xm_status_few():
    return 1   # XM_O_FEW_ITERATIONS


def test_orchestrate_suite_shaped():
    """200 Monte-Carlo-drawn profiles (the paper's model/optimizer/batch mix)."""
    p = C.batch(C.suite_cells(200))
    d = xm.DeviceProfiles.from_host(p)
    cls, seq, rec, wb = xm.orchestrate(d, wire=False)
    cls = cls.cpu().numpy()
    seq = seq.cpu().numpy().view(np.uint64)
    for t in range(p.n_traces):
        a, f, s, st, W = p.trace(t)
        b0 = int(p.boff[t])
        ocls, oev = O.orchestrate(a, f, s, W)
        assert (cls[b0:b0 + len(a)] == np.asarray(ocls, np.uint8)).all(), p.names[t]
        ws = int(rec["ws"][t])
        keys = seq[2 * b0:2 * b0 + int(rec["n_events"][t])]
        assert [(ws + int(k >> 32), int((k >> 31) & 1), int(k & 0x7FFFFFFF)) for k in keys] == oev
