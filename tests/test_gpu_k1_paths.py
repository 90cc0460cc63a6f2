"""K1 (XM_ALLOCATED_ONLY: peak allocated bytes as a segmented prefix-scan/max,
PAPER.md:256 (i), 263) through each of its three kernels -- K1c
(contiguous chunks streamed by TMA, the default), K1t (one CTA per trace) and
the flat path -- vs the oracle, bit-exact on peak_allocated, its first index
and events_done. The batches aim at K1c's seams: traces crossing tile and
chunk boundaries (one trace spans hundreds of chunks, whole chunks without a
trace start), more than 32 trace starts in one tile, one-event and empty
traces, event counts that are not a multiple of the 16-event TMA row, and
batches smaller than one row."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2510_21048_b200 as xm
from gpu_util import assert_parity, oracle_run
from workloads import concat, fuzz, suites
from workloads.trace import TraceBuilder

FIELDS = ["peak_allocated", "peak_allocated_idx", "events_done"]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _random_trace(tb, rng, n, bid, p_free=0.46, max_bytes=1 << 22):
    live = []
    for _ in range(n):
        if live and rng.random() < p_free:
            tb.free(live.pop(int(rng.integers(0, len(live)))))
        else:
            tb.alloc(bid, int(rng.integers(1, max_bytes)))
            live.append(bid)
            bid += 1
    return bid


def _seams_batch(long_len=700_000):
    rng = np.random.default_rng(77)
    tb = TraceBuilder()
    bid = 0
    bid = _random_trace(tb, rng, long_len, bid)            # crosses many chunks
    tb.end_trace()
    for n in [2047, 2048, 2049, 4095, 4097, 30000]:        # around the 2048-event tile
        bid = _random_trace(tb, rng, n, bid)
        tb.end_trace()
    # the peak reached early and then again exactly, many times (first index wins)
    ids = []
    for i in range(3000):
        tb.alloc(bid, 512)
        ids.append(bid)
        bid += 1
    for k in range(6000):
        tb.free(ids.pop())
        tb.alloc(bid, 512)
        ids.append(bid)
        bid += 1
    for i in ids:
        tb.free(i)
    tb.end_trace()
    for _ in range(150):                                   # one-event traces: > 32 starts in a tile
        tb.alloc(bid, int(rng.integers(1, 1 << 20)))
        bid += 1
        tb.end_trace()
    for _ in range(5):                                     # empty traces
        tb.end_trace()
    for n in [2, 3, 5, 7]:
        bid = _random_trace(tb, rng, n, bid)
        tb.end_trace()
    tb.alloc(bid, 3)                                       # total not a multiple of 16
    tb.end_trace()
    return concat([tb.build(), fuzz.spec1_corpus(300, 900, salt=41), suites.config1()])


def _run(b, path, packed):
    old = os.environ.get("XM_K1")
    os.environ["XM_K1"] = path
    try:
        tr = xm.load_traces(b.bytes, b.tag, b.off)
        dev = tr.to_device(packed=packed)
        h, _ = xm.peaks(xm.simulate_batch(dev, xm.Config(mode=1)))
    finally:
        if old is None:
            del os.environ["XM_K1"]
        else:
            os.environ["XM_K1"] = old
    return h


@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("path", ["c", "t", "f"])
def test_k1_paths_seams(path, packed):
    b = _seams_batch()
    h = _run(b, path, packed)
    assert_parity(b, h, oracle_run(b), fields=FIELDS)


@pytest.mark.parametrize("n_events", [1, 5, 15, 16, 17, 33])
def test_k1c_tiny_batches(n_events):
    """Fewer events than one TMA row, or a partial last row: K1c reads them
    from global memory."""
    rng = np.random.default_rng(n_events)
    tb = TraceBuilder()
    bid = 0
    left = n_events
    while left > 0:
        n = int(min(left, rng.integers(1, 6)))
        bid = _random_trace(tb, rng, n, bid)
        tb.end_trace()
        left -= n
    tb.end_trace()                                         # and an empty one
    b = tb.build()
    for packed in (False, True):
        h = _run(b, "c", packed)
        assert_parity(b, h, oracle_run(b), fields=FIELDS)


def test_k1c_config4():
    """The bench's K1 workload (config 4, 5209 traces), every trace."""
    b = suites.config4()
    b = type(b)(b.bytes, b.tag, b.off, np.full(b.n_traces, np.iinfo(np.uint64).max, np.uint64), b.names)
    h = _run(b, "c", True)
    assert_parity(b, h, oracle_run(b, parallel=True), fields=FIELDS)


@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("path", ["c", "t", "f"])
def test_k1_paths_roundup_divisions(path, packed):
    """The NEXT-4 rounding variant (torch roundup_power2_divisions:4, reading
    Q20) through each K1 kernel's division path (kDiv), vs the oracle."""
    b = concat([_seams_batch(long_len=150_000), fuzz.small_size_corpus(200, 600, salt=43)])
    old = os.environ.get("XM_K1")
    os.environ["XM_K1"] = path
    try:
        tr = xm.load_traces(b.bytes, b.tag, b.off)
        dev = tr.to_device(packed=packed)
        h, _ = xm.peaks(xm.simulate_batch(dev, xm.Config(mode=1, roundup_power2_divisions=4)))
    finally:
        if old is None:
            del os.environ["XM_K1"]
        else:
            os.environ["XM_K1"] = old
    assert_parity(b, h, oracle_run(b, div=4), fields=FIELDS)


@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("path", ["c", "t"])
def test_k1_paths_large_requests(path, packed):
    """Requests around 2^31, 2^35 and up to 2^39 bytes, so K1c's common tiles
    take each of its arithmetic tiers (32-bit warp scan, 32-bit lane sums with
    a 64-bit warp scan, all 64-bit) and mix them across the warps of a chunk."""
    rng = np.random.default_rng(91)
    tb = TraceBuilder()
    bid = 0
    for top in [1 << 22, (1 << 31) + 5, 1 << 33, (1 << 35) + 7, 1 << 39]:
        for _ in range(6):
            bid = _random_trace(tb, rng, int(rng.integers(3000, 9000)), bid, max_bytes=top)
            tb.end_trace()
    b = concat([tb.build(), suites.config1()])
    h = _run(b, path, packed)
    assert_parity(b, h, oracle_run(b), fields=FIELDS)
