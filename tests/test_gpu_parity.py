"""CUDA path (libxmem.so, through the C-ABI) vs the oracle, bit-exact on every
result field of every trace. Integer path: the bar is exact equality."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle
import paper_2510_21048_b200 as xm
from gpu_util import COMPARE, assert_parity, gpu_run, oracle_run
from workloads import concat, fuzz, hand, suites
from workloads.trace import TraceBuilder


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _check(batch, cfg=None, strict=1):
    h, _ = gpu_run(batch, cfg)
    o = oracle_run(batch, strict=strict, parallel=batch.n_events > 2_000_000)
    assert_parity(batch, h, o)
    return h


def test_hand_traces(golden):
    named = hand.all_named()
    b = concat(list(named.values()))
    h = _check(b)
    names = list(named)
    for name, g in golden.items():
        t = names.index(name)
        for k, v in g["expect"].items():
            if k in COMPARE:
                assert int(h[k][t]) == v, (name, k)


def test_spec1_fuzz_corpus():
    _check(fuzz.spec1_corpus(1000, 1000, salt=1))


def test_small_pool_corpus():
    _check(fuzz.small_size_corpus(400, 600, salt=2))


def test_capacity_corpus_reclaim_and_oom():
    b = fuzz.capacity_corpus(400, 800, salt=3)
    h = _check(b)
    assert (h["status"] == 1).sum() > 20 and (h["n_seg_release"] > 0).sum() > 20


def test_spec_split_variant():
    b = fuzz.spec1_corpus(200, 600, salt=4)
    _check(b, xm.Config(large_split_strict=0), strict=0)


def test_fragmentation_stress_spills_to_global_arena():
    # 2048 free holes outgrow the initial free-list guess (restart in a 4x
    # region); with a 16 KB heap the state cannot live in shared memory at all
    # (global arena path)
    b = concat([fuzz.fragmentation_stress(), fuzz.fragmentation_stress(8192, 1024, "frag2")])
    _check(b, xm.Config(smem_per_warp=16384, warps_per_cta=1))
    _check(b)


@pytest.mark.parametrize("spw,wpc", [(4096, 1), (8192, 2), (24576, 4), (49152, 8)])
def test_launch_geometries(spw, wpc):
    b = concat([fuzz.spec1_corpus(150, 800, salt=7), fuzz.capacity_corpus(50, 500, salt=8)])
    _check(b, xm.Config(smem_per_warp=spw, warps_per_cta=wpc))


def test_edge_cases():
    tb = TraceBuilder()
    tb.end_trace()                                    # empty
    tb.alloc(0, 1).end_trace()                        # open trace, one event
    tb.alloc(0, (1 << 40) - 1).end_trace()            # largest request
    tb.alloc(0, 3 << 30).free(0).alloc(1, 3 << 30).end_trace(capacity=4 << 30)
    tb.alloc(0, 5 << 30).end_trace(capacity=4 << 30)  # oversize request -> OOM at 0
    for s in range(16):                               # 16 streams
        tb.alloc(s, 1000 + s, stream=s)
    for s in range(16):
        tb.free(s, stream=s)
    tb.end_trace()
    for i in range(70):                               # ragged tile tail: 70 events
        tb.alloc(i, 512 * (i + 1))
    tb.end_trace()
    _check(tb.build())


def test_wide_layout_saturated_keys():
    """Free blocks of >= 2^27 units (64 GiB): the WIDE layout's best-fit key
    saturates, so the winner is chosen by the exact (size, addr) compare
    (replay.cu best_fit_exact). Covers distinct saturated sizes, equal
    saturated sizes in different segments (lowest address wins, reading Q4),
    a request whose candidates mix saturated and exact keys, reclamation of a
    saturated segment, and frees that merge into saturated blocks."""
    G = 1 << 30
    tb = TraceBuilder()
    # distinct saturated sizes, listed larger-first in the free list
    tb.alloc(0, 70 * G).alloc(1, 66 * G).free(0).free(1).alloc(2, 65 * G).alloc(3, 69 * G)
    tb.free(2).alloc(4, 66 * G - 4096).free(3).free(4).alloc(5, 67 * G).end_trace()
    # equal saturated sizes in different segments: lowest address wins
    tb.alloc(0, 68 * G).alloc(1, 68 * G).free(1).free(0).alloc(2, 67 * G).alloc(3, 67 * G)
    tb.free(2).free(3).alloc(4, 68 * G).end_trace()
    # mixed: an exact key (1 GiB) beats the saturated one; then only saturated fit
    tb.alloc(0, 70 * G).alloc(1, G).free(0).free(1).alloc(2, 512 << 20).alloc(3, 2 * G)
    tb.alloc(4, 3 * G).free(3).alloc(5, 600 << 20).free(2).free(4).free(5).end_trace()
    # reclamation with a saturated whole-segment free block (capacity 200 GiB)
    tb.alloc(0, 100 * G).free(0).alloc(1, 150 * G).alloc(2, 40 * G).free(1).alloc(3, 120 * G)
    tb.end_trace(capacity=200 * G)
    # splits of saturated blocks into many pieces, then coalescing back
    tb.alloc(0, 80 * G).free(0)
    for i in range(1, 9):
        tb.alloc(i, 9 * G + 512 * i)
    for i in (2, 4, 6, 8, 1, 3, 5, 7):
        tb.free(i)
    tb.alloc(9, 79 * G).end_trace()
    b = tb.build()
    h = _check(b)
    assert (h["status"][:3] == 0).all() and h["n_seg_release"][3] > 0


def test_config1_mlp():
    _check(suites.config1())


def test_config2_resnet50_sweep():
    _check(suites.config2())


def test_config3_bert_gpt2_streams():
    _check(suites.config3())


def test_config4_full_suite():
    """BASELINE configs[3] at full size (5209 traces) in the bench's launch config."""
    b = suites.config4()
    h = _check(b)
    assert (h["status"] == 2).sum() == 0


@pytest.mark.parametrize("mode", ["auto", "direct", "stream", "copy", "env-stream", "env-no-stream"])
def test_host_entry_point_matches_device_path(mode, monkeypatch):
    """xm_simulate_host with each event-input mode (xm_config.host_input, or
    the env override: the events read in place from the page-locked host array
    by the replaying warps, chunked copies under the replay, one copy first)
    gives the device path's results, which are oracle-checked."""
    cfg = xm.Config(host_input={"direct": 1, "stream": 2, "copy": 3}.get(mode, 0))
    if mode == "env-stream":
        monkeypatch.setenv("XM_HOST_INPUT", "stream")
    if mode == "env-no-stream":
        monkeypatch.setenv("XM_NO_STREAM", "1")
    b = concat([fuzz.capacity_corpus(100, 400, salt=9), suites.config1(), suites.config3()])
    tr = xm.load_traces(b.bytes, b.tag, b.off)
    assert tr.packed is not None
    cap = b.capacity
    h_host, _ = xm.simulate_host(tr, cfg, capacity=cap)
    h_dev, _ = gpu_run(b)
    assert (h_host == h_dev).all()


def test_host_entry_point_without_packed_form():
    """An id space of 2^18 or more has no packed form: xm_simulate_host falls
    back to streaming the 12-byte events (bytes + tag), oracle-checked."""
    tb = TraceBuilder()
    n = (1 << 18) + 40
    for i in range(n):
        tb.alloc(i, 512 * (1 + i % 7))
    for i in range(n):
        tb.free(i)
    tb.end_trace()
    b = concat([tb.build(), suites.config1()])
    tr = xm.load_traces(b.bytes, b.tag, b.off)
    assert tr.packed is None
    h_host, _ = xm.simulate_host(tr, xm.Config())
    assert_parity(b, h_host, oracle_run(b))


def test_host_input_rejects_unknown_mode():
    b = suites.config1()
    tr = xm.load_traces(b.bytes, b.tag, b.off)
    with pytest.raises(xm.XMemError):
        xm.simulate_host(tr, xm.Config(host_input=7))


def test_allocated_only_mode():
    b = concat([fuzz.spec1_corpus(300, 1000, salt=10), suites.config2(), suites.config1()])
    h, _ = gpu_run(b, xm.Config(mode=1))
    o = oracle_run(b)
    assert_parity(b, h, o, fields=["peak_allocated", "peak_allocated_idx", "events_done"])


def test_allocated_only_mode_long_traces():
    """Traces above 65536 events take K1's flat segmented-scan path (shorter
    batches take the trace-per-CTA path tested above)."""
    tb = TraceBuilder()
    rng = np.random.default_rng(5)
    live = []
    for i in range(90_000):
        if live and rng.random() < 0.45:
            tb.free(live.pop(int(rng.integers(0, len(live)))))
        else:
            tb.alloc(i, int(rng.integers(1, 1 << 22)))
            live.append(i)
    tb.end_trace()
    b = concat([tb.build(), fuzz.spec1_corpus(200, 900, salt=12), suites.config1()])
    h, _ = gpu_run(b, xm.Config(mode=1))
    o = oracle_run(b)
    assert_parity(b, h, o, fields=["peak_allocated", "peak_allocated_idx", "events_done"])


def _stepped_traces():
    """Traces around multiples of K1t's step (1024 events: 4 warps x 32 lanes x
    8) up to the trace-per-CTA limit (65536), with first-argmax ties across
    steps and peaks on step boundaries."""
    tb = TraceBuilder()
    rng = np.random.default_rng(21)
    bid = 0
    for n in [4095, 4096, 4097, 8191, 8192, 8193, 12289, 20000, 40000, 65536]:
        live = []
        for _ in range(n):
            if live and rng.random() < 0.47:
                tb.free(live.pop(int(rng.integers(0, len(live)))))
            else:
                tb.alloc(bid, int(rng.integers(1, 1 << 21)))
                live.append(bid)
                bid += 1
        tb.end_trace()
    # the peak reached early and again, exactly, many times later (also at the
    # last event of a step and the first of the next): the first must win
    for first in [100, 4095, 4096]:
        ids = []
        for i in range(first + 1):
            tb.alloc(bid, 512)
            ids.append(bid)
            bid += 1
        k = 0
        while len(ids) > 1 and k < 5000:
            tb.free(ids.pop())
            tb.alloc(bid, 512)
            ids.append(bid)
            bid += 1
            k += 1
        for i in ids:
            tb.free(i)
        tb.end_trace()
    return tb.build()


@pytest.mark.parametrize("packed", [False, True])
def test_allocated_only_mode_stepped_traces(packed):
    b = concat([_stepped_traces(), fuzz.spec1_corpus(100, 900, salt=13), suites.config1()])
    tr = xm.load_traces(b.bytes, b.tag, b.off)
    dev = tr.to_device(packed=packed)
    h, _ = xm.peaks(xm.simulate_batch(dev, xm.Config(mode=1)))
    o = oracle_run(b)
    assert_parity(b, h, o, fields=["peak_allocated", "peak_allocated_idx", "events_done"])


def test_heap_page_handoffs_under_contention():
    """The shared-memory heap's page hand-offs between warps (FIFO admission,
    free-list growth into pages another warp just released, release on trace
    end: fenced atomics on the page bitmap, replay.cu heap_*) under heavy
    contention -- 16 warps on heaps of 6-24 KB per warp, traces of very
    different footprints -- repeated; every run bit-exact vs the oracle, and
    the contended paths provably taken (the kernel's own counters: admission
    waits on the small heaps, free-list growths on the larger ones)."""
    b = concat([fuzz.spec1_corpus(600, 1000, salt=31), fuzz.small_size_corpus(300, 600, salt=32),
                fuzz.capacity_corpus(200, 800, salt=33), fuzz.fragmentation_stress(3000, 512, "fr")])
    o = oracle_run(b)
    tr = xm.load_traces(b.bytes, b.tag, b.off)
    dev = tr.to_device(capacity=b.capacity)
    waits = grows = 0
    for spw in (3072, 6144, 12288, 24576):
        cfg = xm.Config(smem_per_warp=spw, warps_per_cta=16)
        for _ in range(3):
            h, _ = xm.peaks(xm.simulate_batch(dev, cfg))
            assert_parity(b, h, o)
            scr = dev._scratch[(cfg.mode, cfg.smem_per_warp, cfg.warps_per_cta)]
            st = scr[128:160].view(torch.int32).cpu().numpy()     # K2's stats (replay.cu)
            waits += int(st[2])
            grows += int(st[4])
    assert waits > 0 and grows > 0, (waits, grows)


def test_determinism():
    b = fuzz.capacity_corpus(200, 500, salt=11)
    h1, _ = gpu_run(b)
    h2, _ = gpu_run(b)
    assert (h1 == h2).all()


def test_summary_eq1():
    b = hand.h7()
    tr = xm.load_traces(b.bytes, b.tag, b.off)
    dev = tr.to_device(capacity=b.capacity)
    res = xm.simulate_batch(dev)
    _, s = xm.peaks(res)
    assert s["n_oom"] == 1 and s["n_predicted_oom"] == 1
    b2 = hand.h4("late")   # 196 MiB peak; Eq. 1 strict at M_max = 196 MiB
    tr2 = xm.load_traces(b2.bytes, b2.tag, b2.off)
    r2 = xm.simulate_batch(tr2.to_device())
    assert xm.peaks(r2, capacity_for_eq1=196 << 20)[1]["n_predicted_oom"] == 0
    assert xm.peaks(r2, capacity_for_eq1=(196 << 20) - 1)[1]["n_predicted_oom"] == 1


def test_memory_curve_output():
    """per-event (allocated, allocated blocks, reserved) rows
    ("the full series can optionally be output")
    equal the oracle's curve for every processed event."""
    b = concat([fuzz.spec1_corpus(60, 600, salt=41), fuzz.capacity_corpus(40, 500, salt=42),
                suites.config1(), hand.h7(), fuzz.fragmentation_stress()])
    tr = xm.load_traces(b.bytes, b.tag, b.off)
    dev = tr.to_device(capacity=b.capacity)
    curve = torch.zeros((b.n_events, 3), dtype=torch.int64, device="cuda")
    res = xm.simulate_batch(dev, xm.Config(), curve=curve)
    h, _ = xm.peaks(res)
    cv = curve.cpu().numpy().view(np.uint64)
    for t in range(b.n_traces):
        by, tg = b.trace(t)
        o, oc = oracle.simulate_trace(by, tg, int(b.capacity[t]), curve=True)
        n = o["events_done"]
        a, z = tr.span(t)                                  # rows in stored order
        assert int(h["events_done"][t]) == n
        assert (cv[a:a + n] == oc[:n]).all(), (b.names[t], np.flatnonzero((cv[a:a + n] != oc[:n]).any(1))[:3])
        assert (cv[a + n:z] == 0).all()                    # unprocessed rows untouched


# ---- NEXT-4 allocator variants (oracle pins: tests/test_oracle_variants.py) ----
@pytest.mark.parametrize("div", [2, 4, 8])
def test_variant_roundup_power2_divisions(div):
    b = concat([fuzz.spec1_corpus(300, 800, salt=90 + div), fuzz.small_size_corpus(100, 500, salt=95),
                fuzz.capacity_corpus(100, 500, salt=96), suites.config3().subset([0, 30])])
    h, _ = gpu_run(b, xm.Config(roundup_power2_divisions=div))
    assert_parity(b, h, oracle_run(b, div=div))


def test_variant_roundup_allocated_only_mode():
    b = concat([fuzz.spec1_corpus(300, 1000, salt=97), suites.config2().subset([0, 31])])
    h, _ = gpu_run(b, xm.Config(mode=1, roundup_power2_divisions=4))
    assert_parity(b, h, oracle_run(b, div=4),
                  fields=["peak_allocated", "peak_allocated_idx", "events_done"])


def test_variant_d3_largest_first_reclaim(golden):
    b = concat([hand.h8(), fuzz.capacity_corpus(400, 800, salt=98)])
    cfg = xm.Config(reclaim_policy=1)
    h, _ = gpu_run(b, cfg)
    o = oracle_run(b, reclaim=1)
    assert_parity(b, h, o)
    assert (int(h["n_seg_release"][0]), int(h["final_reserved"][0])) == (1, 14 << 20)
    h2, _ = gpu_run(b, xm.Config(reclaim_policy=1, roundup_power2_divisions=4))
    assert_parity(b, h2, oracle_run(b, reclaim=1, div=4))
    # the global-arena (wide) layout takes the same variant paths
    h3, _ = gpu_run(b, xm.Config(reclaim_policy=1, smem_per_warp=4096, warps_per_cta=1))
    assert_parity(b, h3, o)


# ---- NEXT-4: torch max_split_size_mb / garbage_collection_threshold (Q26, Q27) ----
def _knob_corpus():
    import test_oracle_variants as V
    M = 1 << 20
    hands = [V._one(lambda t: t.alloc(0, 100 * M).free(0).alloc(1, 90 * M).free(1).alloc(2, 30 * M)
                    .alloc(3, 70 * M), oracle.UNLIMITED),
             V._one(lambda t: t.alloc(0, 100 * M).alloc(1, 30 * M).alloc(2, M).free(0).free(1)
                    .free(2).alloc(3, 70 * M), 180 * M),
             V._one(lambda t: t.alloc(0, 66 * M).alloc(1, 70 * M).alloc(2, 30 * M).free(0).free(1)
                    .free(2).alloc(3, 120 * M), 200 * M),
             V._one(lambda t: t.alloc(0, 200 * M).alloc(1, 150 * M).alloc(2, 120 * M).alloc(3, 60 * M)
                    .free(0).free(2).alloc(4, 110 * M).free(4).alloc(5, 100 * M).free(5)
                    .alloc(6, 300 * M), 1000 * M)]
    from workloads.trace import from_arrays
    caps = [oracle.UNLIMITED, 180 * M, 200 * M, 1000 * M]
    return concat([from_arrays(by, tg, c) for (by, tg), c in zip(hands, caps)]
                  + [fuzz.spec1_corpus(300, 800, salt=110), fuzz.capacity_corpus(400, 800, salt=111),
                     fuzz.small_size_corpus(100, 500, salt=112), suites.config3().subset([0, 30])])


@pytest.mark.parametrize("msplit,gc", [(21 << 20, 0.0), (32 << 20, 0.0), (64 << 20, 0.0),
                                       (None, 0.3), (None, 0.6), (None, 0.9), (24 << 20, 0.5)])
def test_variant_torch_knobs(msplit, gc):
    b = _knob_corpus()
    cfg = xm.Config(garbage_collection_threshold=gc,
                    **({"max_split_size": msplit} if msplit is not None else {}))
    h, _ = gpu_run(b, cfg)
    o = oracle_run(b, msplit=msplit, gc=gc)
    assert_parity(b, h, o)
    # the knobs change the replay on this corpus (not a vacuous comparison)
    assert (o["peak_reserved"] != oracle_run(b)["peak_reserved"]).any()
    # the global-arena (wide) layout and free-list growth take the same paths
    h2, _ = gpu_run(b, xm.Config(smem_per_warp=4096, warps_per_cta=1, garbage_collection_threshold=gc,
                                 **({"max_split_size": msplit} if msplit is not None else {})))
    assert_parity(b, h2, o)


def test_variant_torch_knobs_config4():
    """Both knobs on the full config-4 suite (its Monte-Carlo half has finite
    capacities, so GC and release_available fire on realistic traces)."""
    b = suites.config4()
    cfg = xm.Config(max_split_size=64 << 20, garbage_collection_threshold=0.6)
    h, _ = gpu_run(b, cfg)
    assert_parity(b, h, oracle_run(b, parallel=True, msplit=64 << 20, gc=0.6))


def test_variant_config_validation():
    b = hand.h7()
    with pytest.raises(xm.XMemError):
        gpu_run(b, xm.Config(roundup_power2_divisions=3))
    with pytest.raises(xm.XMemError):
        gpu_run(b, xm.Config(reclaim_policy=7))
    with pytest.raises(xm.XMemError):
        gpu_run(b, xm.Config(garbage_collection_threshold=1.0))
    with pytest.raises(xm.XMemError):
        gpu_run(b, xm.Config(max_split_size=1000))


def test_packed_event_format():
    """The compact 8-byte events (xm_batch.packed, what xm_simulate_host uploads)
    give the same results as bytes + tag, for K2 (plain, variants, curve) and K1."""
    b = concat([fuzz.spec1_corpus(300, 800, salt=70), fuzz.capacity_corpus(100, 500, salt=71),
                suites.config3().subset([0, 43]), hand.h7()])
    tr = xm.load_traces(b.bytes, b.tag, b.off)
    dp = tr.to_device(capacity=b.capacity, packed=True)
    h, _ = xm.peaks(xm.simulate_batch(dp))
    assert_parity(b, h, oracle_run(b))
    h2, _ = xm.peaks(xm.simulate_batch(dp, xm.Config(reclaim_policy=1, roundup_power2_divisions=4)))
    assert_parity(b, h2, oracle_run(b, reclaim=1, div=4))
    h3, _ = xm.peaks(xm.simulate_batch(dp, xm.Config(smem_per_warp=4096, warps_per_cta=1)))
    assert_parity(b, h3, oracle_run(b))
    d1 = tr.to_device(packed=True)
    k1, _ = xm.peaks(xm.simulate_batch(d1, xm.Config(mode=1)))
    assert_parity(b, k1, oracle_run(type(b)(b.bytes, b.tag, b.off,
                                            np.full(b.n_traces, oracle.UNLIMITED, np.uint64))),
                  fields=["peak_allocated", "peak_allocated_idx", "events_done"])
