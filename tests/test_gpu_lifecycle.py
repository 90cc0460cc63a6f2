"""NEXT-3 lifecycle reconstruction on the GPU (xm_reconstruct, K5) vs the
oracle (oracle/lifecycle.c): partner and mismatch of every instant and every
per-trace tally bit-exact; the wire trace it defines equal to the oracle's
(bytes, streams; block ids valid: one id per open block, reused only after
its block closes); and its replay (K2) equal to the oracle's replay."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle
import paper_2510_21048_b200 as xm
from gpu_util import COMPARE, assert_parity
from workloads import concat, fuzz, instants, suites
from workloads.trace import Batch

TALLIES = ["n_blocks", "n_orphan", "n_mismatch", "n_persistent", "n_kept", "max_open"]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _edge():
    A = np.uint64
    parts = [
        (np.zeros(0, A), np.zeros(0, np.int64)),                       # empty trace
        (np.array([9], A), np.array([-512])),                          # lone orphan
        (np.array([5, 5, 5, 5], A), np.array([100, 200, -200, -100])),  # stacked in one tile
        (np.array([5, 5], A), np.array([100, -96])),                   # mismatch
        (np.array([7] * 70, A), np.array([64, -64] * 35)),             # one address, 70 instants
    ]
    # 40 distinct addresses allocated, then freed in reverse, spanning tiles
    a = np.arange(40, dtype=A) * 4096 + 0x1000
    parts.append((np.r_[a, a[::-1]], np.r_[np.full(40, 256), np.full(40, -256)]))
    off = np.zeros(len(parts) + 1, np.int64)
    off[1:] = np.cumsum([len(p[0]) for p in parts])
    return instants.Instants(np.concatenate([p[0] for p in parts]).astype(A),
                             np.concatenate([p[1] for p in parts]).astype(np.int64),
                             np.zeros(int(off[-1]), np.uint8), off)


def _corpora():
    return [
        _edge(),
        instants.from_batch(fuzz.spec1_corpus(200, 600, salt=51), salt=1,
                            p_orphan=0.01, p_mismatch=0.01, p_lost=0.02),
        instants.from_batch(concat([suites.config1(), suites.config3().subset([0, 21, 43])]),
                            salt=2, p_orphan=0.002, p_mismatch=0.002, p_lost=0.005),
        instants.from_batch(fuzz.small_size_corpus(100, 500, salt=52), salt=3, p_lost=0.05),
    ]


def _check(ins):
    d = xm.DeviceInstants.from_host(ins.addr, ins.bytes, ins.stream, ins.off)
    partner, mism, rec, wb = xm.reconstruct(d)
    partner = partner.cpu().numpy()
    mism = mism.cpu().numpy()
    wbytes = wb.bytes.cpu().numpy()
    wtag = wb.tag.cpu().numpy().view(np.uint32)
    woff = wb.off.cpu().numpy()
    wnids = wb.n_ids.cpu().numpy().view(np.uint32)
    order = wb.order.cpu().numpy().view(np.uint32)
    assert sorted(order.tolist()) == list(range(ins.n_traces))        # a permutation
    kept = rec["n_kept"].astype(np.int64)
    assert (np.diff(kept[order]) <= 0).all()                          # longest first
    pos = np.empty(ins.n_traces, np.int64)
    pos[order] = np.arange(ins.n_traces)
    o_parts = []
    for t in range(ins.n_traces):
        a, by, st = ins.trace(t)
        z0 = int(ins.off[t])
        p, m, tal = oracle.reconstruct(a, by)
        assert (partner[z0:z0 + len(by)] == p).all(), (t, np.flatnonzero(partner[z0:z0 + len(by)] != p)[:5])
        assert (mism[z0:z0 + len(by)] == m).all(), t
        for k in TALLIES:
            assert int(rec[k][t]) == tal[k], (t, k, int(rec[k][t]), tal[k])
        assert tal["max_open"] <= int(rec["n_ids"][t]) <= tal["max_open"] + 31
        # n_reopened: allocations at an address whose earlier block is still open
        # (brute force over the oracle's pairing)
        open_at, reop = {}, 0
        for j in range(len(by)):
            if by[j] > 0:
                reop += open_at.get(int(a[j]), 0) > 0
                open_at[int(a[j])] = open_at.get(int(a[j]), 0) + 1
            elif by[j] < 0 and p[j] >= 0:
                open_at[int(a[j])] -= 1
        assert int(rec["n_reopened"][t]) == reop, (t, int(rec["n_reopened"][t]), reop)
        ob, ot, kept = oracle.wire_from_partner(by, st, p)
        q = pos[t]
        gb = wbytes[woff[q]:woff[q + 1]]
        gt = wtag[woff[q]:woff[q + 1]]
        assert (gb == ob).all(), t
        assert ((gt >> 28) == (ot >> 28)).all(), t
        # ids: an allocation's id comes back on its own free, never on two open blocks
        gid = gt & 0x0FFFFFFF
        assert (gid < wnids[q]).all() and wnids[q] == rec["n_ids"][t]
        live = {}
        ordinal_to_id = {}
        for j in range(len(gb)):
            o_id = int(ot[j] & 0x0FFFFFFF)          # oracle id = allocation ordinal
            if gb[j] > 0:
                assert int(gid[j]) not in live.values()
                live[o_id] = int(gid[j])
                ordinal_to_id[o_id] = int(gid[j])
            else:
                assert live.pop(o_id) == int(gid[j])
        o_parts.append((ob, ot))
    return wb, o_parts


@pytest.mark.parametrize("k", range(4))
def test_reconstruct_parity(k):
    ins = _corpora()[k]
    wb, o_parts = _check(ins)
    # replay of the reconstructed wire trace == oracle replay of the oracle's
    h, _ = xm.peaks(xm.simulate_batch(wb))
    off = np.zeros(len(o_parts) + 1, np.int64)
    off[1:] = np.cumsum([len(p[0]) for p in o_parts])
    ob = Batch(np.concatenate([p[0] for p in o_parts]), np.concatenate([p[1] for p in o_parts]),
               off, np.full(len(o_parts), oracle.UNLIMITED, np.uint64))
    assert_parity(ob, h, oracle.simulate_batch(ob))


def test_reconstruct_config4_shaped():
    """Instants of 300 config-4 traces (25-model suite shape, ~1.7M instants)."""
    b = suites.config4()
    idx = np.linspace(0, b.n_traces - 1, 300).astype(int)
    ins = instants.from_batch(b.subset(idx), salt=4, p_orphan=0.001, p_mismatch=0.001,
                              p_lost=0.002)
    _check(ins)


def test_out_of_range_instants_are_invalid():
    """an instant with |bytes| >= 2^40 (XM_MAX_REQUEST, the replay's
    bound) is counted in n_invalid and ignored like a zero-byte one, so it can
    never reach k_replay's 32-bit unit arithmetic."""
    A = np.uint64
    big = 1 << 40
    ins = instants.Instants(np.array([5, 6, 6, 5], A), np.array([4096, big, -big, -4096], np.int64),
                            np.zeros(4, np.uint8), np.array([0, 4], np.int64))
    d = xm.DeviceInstants.from_host(ins.addr, ins.bytes, ins.stream, ins.off)
    partner, mism, rec, wb = xm.reconstruct(d)
    assert int(rec["n_invalid"][0]) == 2 and int(rec["n_blocks"][0]) == 1
    assert int(rec["n_kept"][0]) == 2 and int(rec["n_orphan"][0]) == 0
    p = partner.cpu().numpy()
    assert p[0] == 3 and p[3] == 0 and p[1] == -1 and p[2] == -1
    assert wb.bytes[:wb.n_events].cpu().numpy().tolist() == [4096, -4096]


@pytest.mark.parametrize("k", range(4))
def test_reconstruct_smem_variant(monkeypatch, k):
    """XM_K5=smem: the shared-memory pass (and k_reconstruct on the traces it
    cannot hold) gives the same partners, mismatches, tallies, dense ids and
    wire form, checked against the oracle as the default kernel is."""
    monkeypatch.setenv("XM_K5", "smem")
    _check(_corpora()[k])


def test_reconstruct_smem_variant_config4_shaped(monkeypatch):
    """... on config-4-shaped instants, where the longest traces overflow the
    shared-memory budget and take the second pass, and against the default
    kernel output for output."""
    b = suites.config4()
    idx = np.linspace(0, b.n_traces - 1, 300).astype(int)
    ins = instants.from_batch(b.subset(idx), salt=5, p_orphan=0.001, p_mismatch=0.001, p_lost=0.002)
    d = xm.DeviceInstants.from_host(ins.addr, ins.bytes, ins.stream, ins.off)
    p0, m0, r0, _ = xm.reconstruct(d)
    monkeypatch.setenv("XM_K5", "smem")
    p1, m1, r1, _ = xm.reconstruct(d)
    assert (p0.cpu() == p1.cpu()).all() and (m0.cpu() == m1.cpu()).all() and (r0 == r1).all()
    _check(ins)
