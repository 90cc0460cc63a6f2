"""K5 (xm_reconstruct) on config-4-shaped instants: time with and without the
wire output (XM_K5_CTAS caps the concurrency; tooling)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from tools.bench_next import _time, _inst_part
from multiprocessing import Pool
from workloads import instants
cuts = np.linspace(0, 5209, 33).astype(int)
with Pool(min(32, os.cpu_count() or 4)) as pool:
    parts = pool.map(_inst_part, list(zip(cuts[:-1], cuts[1:])))
off = [np.zeros(1, np.int64)]
base = 0
for p in parts:
    off.append(p.off[1:] + base)
    base += p.n_events
ins = instants.Instants(np.concatenate([p.addr for p in parts]), np.concatenate([p.bytes for p in parts]),
                        np.concatenate([p.stream for p in parts]), np.concatenate(off))
d = xm.DeviceInstants.from_host(ins.addr, ins.bytes, ins.stream, ins.off)
import ctypes
scratch = torch.empty(int(xm.lib().xm_reconstruct_scratch_bytes(ctypes.byref(d.c()))), dtype=torch.uint8,
                      device="cuda")
reps = int(os.environ.get("REPS", "5"))
ms_nowire = _time(lambda: xm.reconstruct(d, wire=False, scratch=scratch), reps, torch)
ms_wire = _time(lambda: xm.reconstruct(d, wire=True, scratch=scratch), reps, torch)
print(json.dumps({"ctas": os.environ.get("XM_K5_CTAS", "default"), "instants": ins.n_events,
                  "ms_nowire": ms_nowire, "ms_wire": ms_wire}))
