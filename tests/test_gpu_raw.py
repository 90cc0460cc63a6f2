"""xm_simulate_raw: the caller's raw host arrays validated, renumbered and
replayed on the device (K5 keyed by raw block ids -> wire arrays -> K2). The
results equal the oracle's bit-exactly (and the host loader path's), with
pageable and page-locked inputs; every contract violation xm_load_traces
rejects is rejected here too, naming the same first bad trace."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2510_21048_b200 as xm
from gpu_util import assert_parity, gpu_run, oracle_run
from workloads import concat, fuzz, hand, suites
from workloads.trace import TraceBuilder


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _raw(b, cfg=xm.Config(), pinned=False):
    by, tg, off = b.bytes, b.tag, b.off
    if pinned:
        by = torch.from_numpy(np.ascontiguousarray(by)).pin_memory().numpy()
        tg = torch.from_numpy(np.ascontiguousarray(tg).view(np.int32)).pin_memory().numpy().view(np.uint32)
    cap = b.capacity if (b.capacity != xm.UNLIMITED).any() else None
    h, _ = xm.simulate_raw(by, tg, off, cfg, capacity=cap)
    return h


@pytest.mark.parametrize("pinned", [False, True])
def test_raw_matches_oracle(pinned):
    b = concat(list(hand.all_named().values()) + [
        fuzz.spec1_corpus(400, 900, salt=120), fuzz.capacity_corpus(300, 700, salt=121),
        fuzz.small_size_corpus(100, 500, salt=122), suites.config1(), suites.config3()])
    h = _raw(b, pinned=pinned)
    assert_parity(b, h, oracle_run(b))
    hd, _ = gpu_run(b)
    assert (h == hd).all()


def test_raw_config4_full_and_variants():
    b = suites.config4()
    h = _raw(b, pinned=True)
    assert_parity(b, h, oracle_run(b, parallel=True))
    c = fuzz.capacity_corpus(200, 600, salt=123)
    assert_parity(c, _raw(c, xm.Config(roundup_power2_divisions=4)), oracle_run(c, div=4))
    assert_parity(c, _raw(c, xm.Config(max_split_size=24 << 20, garbage_collection_threshold=0.5)),
                  oracle_run(c, msplit=24 << 20, gc=0.5))


@pytest.mark.parametrize("pinned", [False, True])
def test_raw_edge_cases(pinned):
    tb = TraceBuilder()
    tb.end_trace()                                    # empty
    tb.alloc(7, 1).end_trace()                        # open trace
    tb.alloc(0, (1 << 40) - 1).end_trace()            # largest request
    for i in range(70):                               # ragged tile tail
        tb.alloc(1000 + 3 * i, 512 * (i + 1))
    tb.end_trace()
    for s in range(16):                               # 16 streams; frees on another stream
        tb.alloc(s, 1000 + s, stream=s)
    for s in range(16):
        tb.free(s, stream=(s + 1) % 16)
    tb.end_trace()
    b = tb.build()
    assert_parity(b, _raw(b, pinned=pinned), oracle_run(b))


def _bad(kind):
    """Five traces; trace 3 breaks the contract."""
    from workloads.trace import Batch
    good = [(4096, 1), (100, 2), (-4096, 1), (-100, 2)]
    bad = {"dup": [(100, 5), (200, 5)], "nonlive": [(100, 5), (-100, 6)],
           "size": [(100, 5), (-101, 5)], "zero": [(100, 5), (0, 6)]}[kind]
    traces = [good, good, good, bad, [(10, 1), (-10, 1)]]
    by = np.array([b for t in traces for b, _ in t], np.int64)
    tg = np.array([i for t in traces for _, i in t], np.uint32)
    off = np.zeros(len(traces) + 1, np.int64)
    off[1:] = np.cumsum([len(t) for t in traces])
    return Batch(by, tg, off, np.full(len(traces), xm.UNLIMITED, np.uint64))


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("kind", ["dup", "nonlive", "size", "zero"])
def test_raw_rejects_what_the_loader_rejects(kind, pinned):
    """Also with page-locked input (the chunked DMA + per-trace wait path)."""
    b = _bad(kind)
    with pytest.raises(xm.XMemError) as e1:
        xm.load_traces(b.bytes, b.tag, b.off)
    by, tg = b.bytes, b.tag
    if pinned:
        by = torch.from_numpy(np.ascontiguousarray(by)).pin_memory().numpy()
        tg = torch.from_numpy(np.ascontiguousarray(tg).view(np.int32)).pin_memory().numpy().view(np.uint32)
    with pytest.raises(xm.XMemError) as e2:
        xm.simulate_raw(by, tg, b.off)
    assert e2.value.bad_trace == 3
    assert "trace 3" in str(e1.value) and "trace 3" in str(e2.value)


def test_raw_streamed_equals_in_place(monkeypatch):
    """Page-locked input: the chunked DMA copies (default) and the loader
    reading host memory in place (XM_RAW_INPUT=direct) give the same results,
    on a batch of many short traces (chunks of many traces) and long ones."""
    b = concat([fuzz.spec1_corpus(400, 900, salt=51), suites.config2(), fuzz.capacity_corpus(50, 400, salt=52)])
    h1 = _raw(b, pinned=True)
    monkeypatch.setenv("XM_RAW_INPUT", "direct")
    h2 = _raw(b, pinned=True)
    assert (h1 == h2).all()
    assert_parity(b, h1, oracle_run(b))


def _big_mixed(salt):
    """More traces than the replay has warp slots (148 SMs x 14), so
    xm_simulate_raw overlaps the loader with the replay: short fuzz traces, a
    capacity corpus (OOMs, reclamation) and long training traces."""
    return concat([fuzz.spec1_corpus(1800, 400, salt=salt), fuzz.capacity_corpus(400, 500, salt=salt + 1),
                   suites.config2(), fuzz.small_size_corpus(300, 300, salt=salt + 2)])


@pytest.mark.parametrize("loader_sms", ["1", "17", "48", "100", "147"])
def test_raw_overlapped_replay(monkeypatch, loader_sms):
    """The overlapped path (loader on XM_RAW_LOADER_SMS SMs publishing traces
    as it finishes them, the replay on the rest, then a second replay launch
    on the loader's SMs) equals the oracle and the sequential path
    (XM_RAW_OVERLAP=0), whatever the split."""
    b = _big_mixed(61)
    assert b.n_traces > 148 * 14
    monkeypatch.setenv("XM_RAW_LOADER_SMS", loader_sms)
    h = _raw(b, pinned=True)
    assert xm.last_launch_count() == 3             # loader + two replay launches
    assert_parity(b, h, oracle_run(b, parallel=True))
    monkeypatch.setenv("XM_RAW_OVERLAP", "0")
    assert (_raw(b, pinned=True) == h).all()


@pytest.mark.parametrize("kind", ["dup", "nonlive", "size", "zero"])
def test_raw_overlapped_rejects(kind):
    """A contract violation inside a batch large enough for the overlapped
    path is reported with its trace index, as on the sequential path."""
    b = _big_mixed(71)
    bad = _bad(kind)
    at = 1234
    b = concat([b.subset(range(at)), bad.subset([3]), b.subset(range(at, b.n_traces))])
    with pytest.raises(xm.XMemError) as e:
        _raw(b, pinned=True)
    assert e.value.bad_trace == at
    assert f"trace {at}" in str(e.value)


def test_raw_overlapped_first_call_in_fresh_process():
    """The overlapped path's first call in a process (kernel modules not yet
    loaded: CUDA lazy loading must not stall the concurrently running loader
    and replay)."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, torch, paper_2510_21048_b200 as xm\n"
            "from workloads import suites\n"
            "b = suites.config4()\n"
            "by = torch.from_numpy(b.bytes).pin_memory().numpy()\n"
            "tg = torch.from_numpy(b.tag.view(np.int32)).pin_memory().numpy().view(np.uint32)\n"
            "h, _ = xm.simulate_raw(by, tg, b.off, xm.Config(), capacity=b.capacity)\n"
            "assert xm.last_launch_count() == 3\n"
            "np.save('/tmp/xm_fresh_raw.npy', h)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root, CUDA_MODULE_LOADING="LAZY")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    h = np.load("/tmp/xm_fresh_raw.npy")
    b = suites.config4()
    assert_parity(b, h, oracle_run(b, parallel=True))


def test_raw_overlapped_wide_layout_traces():
    """Traces that leave the shared-memory layout (>= 64 GiB blocks, a 1 TiB
    request) spread through a batch large enough for the overlapped path:
    both replay launches restart them in the global arena, sharing its slots."""
    G = 1 << 30
    tb = TraceBuilder()
    for r in range(40):
        tb.alloc(0, 70 * G).alloc(1, 66 * G).free(0).free(1).alloc(2, 65 * G).alloc(3, 69 * G)
        tb.free(2).alloc(4, 66 * G - 4096).free(3).free(4).alloc(5, 67 * G).end_trace()
        tb.alloc(0, (1 << 40) - 1 - r).alloc(1, 512).free(1).end_trace()
        tb.alloc(0, 100 * G).free(0).alloc(1, 150 * G).alloc(2, 40 * G).free(1).alloc(3, 120 * G)
        tb.end_trace(capacity=200 * G)
    wide = tb.build()
    big = _big_mixed(81)
    parts, step = [], big.n_traces // wide.n_traces
    for i in range(wide.n_traces):
        parts += [big.subset(range(i * step, (i + 1) * step)), wide.subset([i])]
    parts.append(big.subset(range(wide.n_traces * step, big.n_traces)))
    b = concat(parts)
    h = _raw(b, pinned=True)
    assert xm.last_launch_count() == 3
    assert_parity(b, h, oracle_run(b, parallel=True))


def _reused_ids(n_traces, seed):
    """Traces whose raw block ids are reused after their block is freed (the
    contract forbids only the alloc of a LIVE id), with 28-bit ids
    spread over the id space and random streams."""
    rng = np.random.default_rng(seed)
    tb = TraceBuilder()
    for _ in range(n_traces):
        pool = rng.choice(1 << 28, size=int(rng.integers(3, 12)), replace=False)
        live = {}
        for _ in range(int(rng.integers(20, 200))):
            free_ids = [i for i in pool if i not in live]
            if live and (not free_ids or rng.random() < 0.45):
                bid = list(live)[int(rng.integers(len(live)))]
                tb.free(int(bid), stream=int(live.pop(bid)))
            else:
                bid = free_ids[int(rng.integers(len(free_ids)))]
                st = int(rng.integers(0, 3))
                live[bid] = st
                tb.alloc(int(bid), int(rng.integers(1, 64 << 20)), stream=st)
        for bid in list(live):
            tb.free(int(bid), stream=live.pop(bid))
        tb.end_trace()
    return tb.build()


@pytest.mark.parametrize("overlapped", [False, True])
def test_raw_reused_block_ids(monkeypatch, overlapped):
    """Raw ids reused after their free: the loader reopens a closed key (k_load)
    and the replay matches the oracle and the host loader's path; sequential
    and overlapped, and with K5's loader (XM_LOADER=k5)."""
    b = _reused_ids(2300 if overlapped else 300, seed=7 + int(overlapped))
    h = _raw(b, pinned=True)
    assert xm.last_launch_count() == (3 if overlapped else 2)
    assert_parity(b, h, oracle_run(b, parallel=overlapped))
    hd, _ = gpu_run(b)
    assert (h == hd).all()
    monkeypatch.setenv("XM_LOADER", "k5")
    assert (_raw(b, pinned=True) == h).all()


@pytest.mark.parametrize("variant", ["div4", "d3", "knobs"])
def test_raw_overlapped_variants(variant):
    """The allocator variants through the overlapped path (the knobs run the
    separate k_replay<true> instantiation in both replay launches)."""
    b = _big_mixed(91)
    cfg, ora = {"div4": (xm.Config(roundup_power2_divisions=4), dict(div=4)),
                "d3": (xm.Config(reclaim_policy=1), dict(reclaim=1)),
                "knobs": (xm.Config(max_split_size=24 << 20, garbage_collection_threshold=0.5),
                          dict(msplit=24 << 20, gc=0.5))}[variant]
    h = _raw(b, cfg, pinned=True)
    assert xm.last_launch_count() == 3
    assert_parity(b, h, oracle_run(b, parallel=True, **ora))
