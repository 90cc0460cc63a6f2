"""K2's two bounds on config 4: the LPT makespan over the kernel's warp slots
(148 SMs x 14 warps, traces pulled longest-first) vs the average load per slot,
in events. Host-only (no GPU, no oracle)."""
import heapq
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import suites  # noqa: E402

slots = int(sys.argv[1]) if len(sys.argv) > 1 else 148 * 14
n = np.sort(suites.config4().lengths())[::-1]
h = [0] * slots
for x in n:
    heapq.heappush(h, heapq.heappop(h) + int(x))
print(f"traces {len(n)}  events {int(n.sum())}  slots {slots}")
print(f"longest trace {int(n[0])}  LPT makespan {max(h)}  mean per slot {n.sum() / slots:.0f}")
print(f"traces > 10k events: {int((n > 10000).sum())}")
