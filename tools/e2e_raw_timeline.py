"""Where xm_simulate_raw's time goes on config 4: torch.profiler (CUPTI) trace
of one call: the kernels (start, duration), the first and last copy, the
host gaps."""
import os, sys
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
ev = sorted(prof.events(), key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
cuda = [e for e in ev if e.device_type.name == "CUDA"]
cp = [e for e in cuda if "HtoD" in e.name]
ker = [e for e in cuda if "Memcpy" not in e.name and "Memset" not in e.name]
f = lambda x: round((x - t0) / 1e3, 3)
if cp:
    print("H2D copies:", len(cp), "first start", f(cp[0].time_range.start), "last end", f(max(e.time_range.end for e in cp)))
for e in ker:
    print("kernel", e.name[:50], "start", f(e.time_range.start), "end", f(e.time_range.end))
print("last event end", f(max(e.time_range.end for e in cuda)))
