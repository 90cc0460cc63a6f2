"""Where xm_simulate_raw's time goes on config 4: torch.profiler (CUPTI) trace
of one call: the kernels, the copies and the host gaps between them."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from workloads import suites
b = suites.config4()
pin_b = torch.from_numpy(b.bytes).pin_memory().numpy()
pin_t = torch.from_numpy(b.tag.view(np.int32)).pin_memory().numpy().view(np.uint32)
_, ws = xm.simulate_raw(pin_b, pin_t, b.off, xm.Config(), capacity=b.capacity)
_, ws = xm.simulate_raw(pin_b, pin_t, b.off, xm.Config(), capacity=b.capacity, workspace=ws)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    xm.simulate_raw(pin_b, pin_t, b.off, xm.Config(), capacity=b.capacity, workspace=ws)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA" or "Memcpy" in e.name or "cuda" in e.name.lower()]
rows = []
t0 = None
for e in sorted(prof.events(), key=lambda e: e.time_range.start):
    if t0 is None:
        t0 = e.time_range.start
    rows.append((round((e.time_range.start - t0) / 1e3, 3), round((e.time_range.end - e.time_range.start) / 1e3, 3),
                 e.device_type.name, e.name[:60]))
for r in rows:
    if r[1] > 0.02 or r[2] == "CUDA":
        print(r)
