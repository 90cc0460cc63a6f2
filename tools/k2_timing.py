"""Per-trace start/end times of K2 (XM_TIMING build) on a workload."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from paper_2510_21048_b200 import _build
xm._lib = None
_build.LIB = os.path.join(_build.PKG, "libxmem_timing.so")
from workloads import suites
b = suites.config4()
tr = xm.load_traces(b.bytes, b.tag, b.off)
cap = b.capacity if (b.capacity != xm.UNLIMITED).any() else None
dev = tr.to_device("cuda", capacity=cap)
cfg = xm.Config(warps_per_cta=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
out = xm.simulate_batch(dev, cfg); torch.cuda.synchronize()
out = xm.simulate_batch(dev, cfg, out=out); torch.cuda.synchronize()
scr = list(dev._scratch.values())[-1]
T = b.n_traces
tim = scr[-T * 16:].view(torch.int64).cpu().numpy().reshape(T, 2)
t0 = tim[:, 0].min(); st = (tim[:, 0] - t0) / 1e6; en = (tim[:, 1] - t0) / 1e6
L = np.diff(b.off); h, _ = xm.peaks(out); done = h["events_done"].astype(np.int64)
dur = en - st
order = np.argsort(-en)
print(f"makespan {en.max():.3f} ms")
for i in order[:8]:
    print(f"trace {i:5d} {b.names[i][:50]:50s} n={L[i]:6d} done={done[i]:6d} start={st[i]:.3f} end={en[i]:.3f} dur={dur[i]:.3f} ms  ns/event={dur[i]*1e6/max(done[i],1):.0f}")
rate = done / np.maximum(dur, 1e-9) / 1e3
print("per-trace ns/event quantiles", np.quantile(dur * 1e6 / np.maximum(done, 1), [0.1, 0.5, 0.9]))
print("start times quantiles", np.quantile(st, [0, .5, .9, 1]))
busy = dur.sum()
W = 148 * (cfg.warps_per_cta or 14)
print(f"warp-slot utilisation {busy / (en.max() * W) * 100:.1f}% (sum of trace durations / makespan x {W} warps)")
for q in (0.5, 0.8, 0.9, 0.95, 1.0):
    print(f"  {q*100:.0f}% of traces done by {np.quantile(en, q):.3f} ms")
np.savez(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "k2_timing.npz"),
         start=st, end=en, n=L, done=done, n_ids=tr.n_ids[tr.pos].astype(np.int64), names=np.asarray(b.names))
