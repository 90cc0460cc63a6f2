"""Time K2 on a subset of config-4 traces selected by name substring (argv[1])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from workloads import suites
b = suites.config4()
idx = [i for i, n in enumerate(b.names) if sys.argv[1] in n]
b = b.subset(idx)
tr = xm.load_traces(b.bytes, b.tag, b.off)
cap = b.capacity if (b.capacity != xm.UNLIMITED).any() else None
dev = tr.to_device("cuda", capacity=cap)
cfg = xm.Config(warps_per_cta=int(sys.argv[2]) if len(sys.argv) > 2 else 1)
out = xm.simulate_batch(dev, cfg); torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); xm.simulate_batch(dev, cfg, out=out); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
h, _ = xm.peaks(out)
done = h["events_done"].astype(np.int64)
print(f"{sys.argv[1]}: {len(idx)} traces, max len {done.max()}, {min(ts):.3f} ms -> {min(ts)*1e6/done.max():.0f} ns/event on the longest")
