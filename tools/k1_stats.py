"""Time K1 (allocated-only segmented scan) on a workload; print achieved GB/s."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from workloads import suites
wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
rep = int(sys.argv[2]) if len(sys.argv) > 2 else 1
b = suites.CONFIGS[wl]()
if rep > 1:
    from workloads import concat
    b = concat([b] * rep)
tr = xm.load_traces(b.bytes, b.tag, b.off)
dev = tr.to_device("cuda")
cfg = xm.Config(mode=1)
out = xm.simulate_batch(dev, cfg)
torch.cuda.synchronize()
ts = []
reps = int(os.environ.get("REPS", "20"))
for _ in range(10):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _r in range(reps):
        xm.simulate_batch(dev, cfg, out=out)
    e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / reps)
ms = float(np.median(ts))
alg = 8 * b.n_events + 8 * (b.n_traces + 1) + 64 * b.n_traces
print(json.dumps({"path": os.environ.get("XM_K1", "c"), "workload": wl, "rep": rep, "n_events": b.n_events, "ms": ms, "min_ms": min(ts),
                  "GBps": alg / (ms / 1e3) / 1e9, "ev_per_s": b.n_events / (ms / 1e3),
                  "launches": xm.last_launch_count()}))
