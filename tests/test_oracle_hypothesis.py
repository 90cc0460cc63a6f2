"""Property-based pin of the oracle (hypothesis): on small random traces with
random allocator knobs (split strictness, roundup_power2_divisions, reclaim
policy, capacity), the oracle's per-event curve and every result field equal
the independent gap-model brute force (tests/bruteforce.py). No GPU."""
import numpy as np
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import bruteforce
import oracle

MiB = 1 << 20


@st.composite
def traces(draw):
    n_ops = draw(st.integers(1, 120))
    sizes = st.one_of(st.integers(1, 4096), st.integers(4096, 2 * MiB), st.integers(2 * MiB, 40 * MiB))
    live, by, tg = [], [], []
    nxt = 0
    for _ in range(n_ops):
        if live and draw(st.booleans()):
            k = draw(st.integers(0, len(live) - 1))
            bid, size, stream = live.pop(k)
            by.append(-size)
            tg.append(bid | (stream << 28))
        else:
            size = draw(sizes)
            stream = draw(st.integers(0, 2))
            live.append((nxt, size, stream))
            by.append(size)
            tg.append(nxt | (stream << 28))
            nxt += 1
    cap = draw(st.one_of(st.just(oracle.UNLIMITED), st.integers(2, 200).map(lambda m: m * MiB)))
    return np.array(by, np.int64), np.array(tg, np.uint32), cap


@settings(max_examples=300, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(traces(), st.booleans(), st.sampled_from([0, 2, 4, 8]), st.sampled_from([0, 1]))
def test_oracle_equals_bruteforce(tr, strict, div, reclaim):
    by, tg, cap = tr
    cfg = oracle.Config(large_split_strict=int(strict), roundup_power2_divisions=div,
                        reclaim_policy=reclaim)
    o, oc = oracle.simulate_trace(by, tg, cap, cfg=cfg, curve=True, check=True)
    b, bc = bruteforce.simulate(by, tg, cap, strict=strict, div=div, reclaim=reclaim)
    for k, v in b.items():
        assert o[k] == v, (k, o[k], v)
    n = o["events_done"]
    assert oc[:n].tolist() == [list(x) for x in bc[:n]]
