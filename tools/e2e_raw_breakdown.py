"""Time xm_simulate_raw on config 4 (page-locked raw arrays) and, under ncu's
launch list, its kernels; also the plain DMA copy of the raw arrays."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from workloads import suites
b = suites.config4()
cfg = xm.Config()
pin_b = torch.from_numpy(b.bytes).pin_memory().numpy()
pin_t = torch.from_numpy(b.tag).pin_memory().numpy()
capn = b.capacity
_, ws = xm.simulate_raw(pin_b, pin_t, b.off, cfg, capacity=capn)
reps = int(os.environ.get("REPS", "5"))
ts = []
for _ in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    xm.simulate_raw(pin_b, pin_t, b.off, cfg, capacity=capn, workspace=ws)
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
d_b = torch.empty(b.n_events, dtype=torch.int64, device="cuda")
d_t = torch.empty(b.n_events, dtype=torch.int32, device="cuda")
tb = torch.from_numpy(pin_b); tt = torch.from_numpy(pin_t.view(np.int32))
cs = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); d_b.copy_(tb, non_blocking=True); d_t.copy_(tt, non_blocking=True); e1.record()
    torch.cuda.synchronize(); cs.append(e0.elapsed_time(e1))
print(json.dumps({"simulate_raw_ms": ts, "dma_copy_raw_ms": cs, "raw_bytes": 12 * b.n_events}))
