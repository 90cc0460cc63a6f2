"""k_replay reading its packed events from HBM vs straight from the page-locked
host array (the direct input of xm_simulate_host), timed with CUDA events; and
the per-call host overhead of xm_simulate_host on a tiny batch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from workloads import suites

b = suites.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]()
tr = xm.load_traces(b.bytes, b.tag, b.off)
cap = b.capacity if (b.capacity != xm.UNLIMITED).any() else None
dev = tr.to_device("cuda", capacity=cap, packed=True)
cfg = xm.Config()


def kt(d, reps=5):
    out = xm.simulate_batch(d, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); xm.simulate_batch(d, cfg, out=out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return np.median(ts), out


t_hbm, o1 = kt(dev)
host = torch.from_numpy(tr.packed.view(np.int64))       # page-locked, device-mapped (UVA)
dev.packed = host
t_host, o2 = kt(dev)
same = bool((o1.cpu() == o2.cpu()).all())
print(f"kernel events in HBM {t_hbm:.3f} ms, events read from host {t_host:.3f} ms, same={same}")
# e2e call overhead on the same batch
ws = None
for _ in range(3):
    _, ws = xm.simulate_host(tr, cfg, capacity=cap, workspace=ws)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    _, ws = xm.simulate_host(tr, cfg, capacity=cap, workspace=ws)
print(f"xm_simulate_host {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
s = suites.CONFIGS["cfg1"]()
trs = xm.load_traces(s.bytes, s.tag, s.off)
ws = None
for _ in range(3):
    _, ws = xm.simulate_host(trs, cfg, workspace=ws)
t0 = time.perf_counter()
for _ in range(50):
    _, ws = xm.simulate_host(trs, cfg, workspace=ws)
print(f"xm_simulate_host tiny batch {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms")
