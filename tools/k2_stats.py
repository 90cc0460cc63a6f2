"""Run config 4 through K2 with several launch geometries; print time and heap stats."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from workloads import suites
wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
b = suites.CONFIGS[wl]()
tr = xm.load_traces(b.bytes, b.tag, b.off)
cap = b.capacity if (b.capacity != xm.UNLIMITED).any() else None
dev = tr.to_device("cuda", capacity=cap, packed=bool(os.environ.get("PACKED")))
for wpc in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,8,16").split(",")]:
    cfg = xm.Config(warps_per_cta=wpc, smem_per_warp=int(os.environ.get("SPW", "0")))
    out = xm.simulate_batch(dev, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); xm.simulate_batch(dev, cfg, out=out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    scr = list(dev._scratch.values())[-1]
    st = scr[128:160].view(torch.int32).cpu().numpy()
    ev = int(xm.peaks(out)[0]["events_done"].astype(np.int64).sum())
    print(f"spw={cfg.smem_per_warp} wpc={wpc:2d} ms={min(ts):8.2f} ev/s={ev/min(ts)*1e3:.3e} spills={st[0]} arena={st[1]} heap_wait={st[2]} ticket_wait={st[3]} grows={st[4]}", flush=True)
