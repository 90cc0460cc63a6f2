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
