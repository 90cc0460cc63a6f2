"""xMem's pipeline on the GPU (xm.estimate): profiler instants -> lifecycle
reconstruction (K5) -> blocks (xm_blocks_from_instants) -> memory orchestrator
(K6) -> replay (K2), against the same chain of oracles (oracle.reconstruct ->
blocks -> oracle.orchestrator -> oracle.simulate_trace), bit-exact on every
result field; the reconstructed blocks also equal the generator's."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle
import paper_2510_21048_b200 as xm
from gpu_util import COMPARE
from oracle import orchestrator as O
from workloads import cpu_profile as C


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


CELLS = [("mobilenet_v2", "adam", "pos0", 200, False), ("gpt2", "adamw", "pos1", 5, True),
         ("resnet101", "sgd", "pos1", 300, False), ("t5_small", "adafactor", "pos0", 10, False),
         ("vgg16", "rmsprop", "pos1", 200, False), ("bert_base", "adamw", "pos0", 15, True)]


def _oracle_chain(ts, ad, by, st, W, cap):
    part, _, _ = oracle.reconstruct(ad, by)
    al = np.flatnonzero(by > 0)
    a = ts[al]
    f = np.where(part[al] >= 0, ts[np.maximum(part[al], 0)], -1)
    s = by[al]
    sst = st[al]
    cls, ev = O.orchestrate(a, f, s, W)
    wb, wt = O.wire(ev, s, sst)
    r, _ = oracle.simulate_trace(wb, wt, cap)
    return (a, f, s), r


@pytest.mark.parametrize("capacity", [None, 6 << 30])
def test_estimate_pipeline_matches_oracle_chain(capacity):
    p = C.batch(CELLS)
    ts, ad, by, st, off = C.to_instants(p)
    d = xm.DeviceInstants.from_host(ad, by, st, off)
    d_ts = torch.from_numpy(ts).cuda()
    caps = None if capacity is None else np.full(p.n_traces, capacity, np.uint64)
    h, summ, det = xm.estimate(d, d_ts, p.win, p.woff, capacity=caps)
    prof = det["profiles"]
    ga = prof.alloc_ts.cpu().numpy()
    gf = prof.free_ts.cpu().numpy()
    gs = prof.size.cpu().numpy()
    boff = prof.boff.cpu().numpy()
    for t in range(p.n_traces):
        z0, z1 = int(off[t]), int(off[t + 1])
        W = p.win[p.woff[t]:p.woff[t + 1]]
        cap = oracle.UNLIMITED if capacity is None else capacity
        (a, f, s), r = _oracle_chain(ts[z0:z1], ad[z0:z1], by[z0:z1], st[z0:z1], W, cap)
        b0, b1 = int(boff[t]), int(boff[t + 1])
        assert (ga[b0:b1] == a).all() and (gf[b0:b1] == f).all() and (gs[b0:b1] == s).all()
        pa, pf, ps, _, _ = p.trace(t)                 # the generator's own blocks
        assert (a == pa).all() and (f == pf).all() and (s == ps).all()
        for k in COMPARE:
            exp = min(r[k], 65535) if k == "n_free_blocks_end" else r[k]
            assert int(h[k][t]) == exp, (p.names[t], k, int(h[k][t]), exp)
    if capacity is not None:
        assert summ["n_oom"] > 0


def test_estimate_curve_matches_oracle_curve():
    """The pipeline's optional memory-usage curve equals the
    oracle's curve of the same re-timed sequence, event by event."""
    p = C.batch(CELLS[:3])
    ts, ad, by, st, off = C.to_instants(p)
    d = xm.DeviceInstants.from_host(ad, by, st, off)
    h, _, det = xm.estimate(d, torch.from_numpy(ts).cuda(), p.win, p.woff, curve=True)
    wb = det["wire"]
    cv = det["curve"].cpu().numpy().view(np.uint64)
    woff = wb.off.cpu().numpy()
    order = wb.order.cpu().numpy().view(np.uint32)
    pos = np.empty(p.n_traces, np.int64)
    pos[order] = np.arange(p.n_traces)
    for t in range(p.n_traces):
        z0, z1 = int(off[t]), int(off[t + 1])
        W = p.win[p.woff[t]:p.woff[t + 1]]
        part, _, _ = oracle.reconstruct(ad[z0:z1], by[z0:z1])
        al = np.flatnonzero(by[z0:z1] > 0)
        a = ts[z0:z1][al]
        f = np.where(part[al] >= 0, ts[z0:z1][np.maximum(part[al], 0)], -1)
        s = by[z0:z1][al]
        _, ev = O.orchestrate(a, f, s, W)
        wbb, wtt = O.wire(ev, s, st[z0:z1][al])
        r, oc = oracle.simulate_trace(wbb, wtt, curve=True)
        q = pos[t]
        assert (cv[woff[q]:woff[q + 1]] == oc).all(), t


def test_estimate_rejects_traces_without_enough_iterations():
    """a trace with fewer than analysis_iter + 1 iterations has no
    analysis window (an error). estimate() raises instead of
    replaying the empty sequence K6 leaves for it as a 0-byte peak."""
    p = C.batch(CELLS[:2])
    ts, ad, by, st, off = C.to_instants(p)
    d = xm.DeviceInstants.from_host(ad, by, st, off)
    n_iter = int(np.diff(p.woff).min())
    with pytest.raises(xm.XMemError, match="fewer than analysis_iter"):
        xm.estimate(d, torch.from_numpy(ts).cuda(), p.win, p.woff, analysis_iter=n_iter)
