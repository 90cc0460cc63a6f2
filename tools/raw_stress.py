"""Stress of xm_simulate_raw's overlapped path (concurrent copies, loader and
replay): N calls on config 4 and on a GPU-filling fuzz batch with capacities,
every result compared with the device path's (xm_simulate_batch on the
host-loaded batch). Prints the number of mismatching calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from workloads import concat, fuzz, suites
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for name, b in [("config4", suites.config4()),
                ("fuzz", concat([fuzz.spec1_corpus(2000, 300, salt=5), fuzz.capacity_corpus(600, 400, salt=6)]))]:
    tr = xm.load_traces(b.bytes, b.tag, b.off)
    cap = b.capacity if (b.capacity != xm.UNLIMITED).any() else None
    ref, _ = xm.peaks(xm.simulate_batch(tr.to_device(capacity=cap)))
    pb = torch.from_numpy(np.ascontiguousarray(b.bytes)).pin_memory().numpy()
    pt = torch.from_numpy(np.ascontiguousarray(b.tag).view(np.int32)).pin_memory().numpy().view(np.uint32)
    ws, bad = None, 0
    for i in range(n):
        h, ws = xm.simulate_raw(pb, pt, b.off, xm.Config(), capacity=cap, workspace=ws)
        bad += int(not (h == ref).all())
    print(f"{name}: {n} overlapped calls (launches {xm.last_launch_count()}), {bad} with results != device path",
          flush=True)
