"""xm_simulate_host wall time per event-input mode (XM_HOST_INPUT) on config 4."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from workloads import suites

b = suites.config4()
tr = xm.load_traces(b.bytes, b.tag, b.off)
cap = b.capacity if (b.capacity != xm.UNLIMITED).any() else None
cfg = xm.Config()
ws = None
ref = None
MODES = ("direct", "stream", "copy")    # xm_simulate_host event inputs (capi.cu)
for m in (sys.argv[1:] or os.environ.get("XM_E2E_MODES", "direct stream copy").split()):
    if m not in MODES:
        raise SystemExit(f"unknown host-input mode {m!r}; one of {MODES}")
    os.environ["XM_HOST_INPUT"] = m
    for _ in range(3):
        h, ws = xm.simulate_host(tr, cfg, capacity=cap, workspace=ws)
    ref = h if ref is None else ref
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        h, ws = xm.simulate_host(tr, cfg, capacity=cap, workspace=ws)
        ts.append(time.perf_counter() - t0)
    print(f"{m:7s} median {np.median(ts) * 1e3:.3f} ms  min {min(ts) * 1e3:.3f} ms  same={(h == ref).all()}",
          flush=True)
