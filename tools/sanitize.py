"""Small runs of every kernel path, for compute-sanitizer (memcheck / racecheck /
synccheck): python tools/sanitize.py  (run under compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2510_21048_b200 as xm
from workloads import concat, cpu_profile, fuzz, hand, instants, mc5, suites

b = concat([fuzz.spec1_corpus(12, 300, salt=1), fuzz.capacity_corpus(6, 300, salt=3),
            suites.config1(), hand.h7(), hand.h8()])
tr = xm.load_traces(b.bytes, b.tag, b.off)
dev = tr.to_device(capacity=b.capacity)
curve = torch.zeros((b.n_events, 3), dtype=torch.int64, device="cuda")
xm.peaks(xm.simulate_batch(dev, curve=curve))                                  # K2 + curve
xm.peaks(xm.simulate_batch(dev, xm.Config(reclaim_policy=1, roundup_power2_divisions=4)))
xm.peaks(xm.simulate_batch(dev, xm.Config(smem_per_warp=4096, warps_per_cta=1)))  # wide arena
xm.simulate_host(tr, xm.Config(), capacity=b.capacity)                         # e2e, direct input
xm.simulate_host(tr, xm.Config(host_input=2), capacity=b.capacity)             # e2e, streamed copies
dev_pk = tr.to_device(capacity=b.capacity, packed=True)
xm.peaks(xm.simulate_batch(dev_pk))                                            # K2, packed events
dev1 = tr.to_device()
xm.peaks(xm.simulate_batch(dev1, xm.Config(mode=1)))                           # K1t
tb = fuzz.spec1_corpus(1, 1000, salt=5)
big = concat([tb] * 70)
long = concat([fuzz.fragmentation_stress(40000, 1024, "long")])                # > 65536 events
trl = xm.load_traces(long.bytes, long.tag, long.off)
xm.peaks(xm.simulate_batch(trl.to_device(), xm.Config(mode=1)))               # K1c (auto: > 65536)
os.environ["XM_K1"] = "c"
xm.peaks(xm.simulate_batch(dev1, xm.Config(mode=1)))                           # K1c, short traces
xm.peaks(xm.simulate_batch(tr.to_device(packed=True), xm.Config(mode=1)))      # K1c, packed
os.environ["XM_K1"] = "f"
xm.peaks(xm.simulate_batch(trl.to_device(), xm.Config(mode=1)))               # K1 flat
del os.environ["XM_K1"]
pin_b = torch.from_numpy(b.bytes).pin_memory().numpy()
pin_t = torch.from_numpy(b.tag.view(np.int32)).pin_memory().numpy().view(np.uint32)
xm.simulate_raw(pin_b, pin_t, b.off, xm.Config(), capacity=b.capacity)        # raw: DMA chunks + loader
d = mc5.describe(np.arange(50))
pool = xm.Templates(*mc5.template_pool())
xm.peaks(xm.simulate_batch(xm.expand_templates(pool, d["tpl"], d["b"], d["seed"],
                                               mc5.SWAP_THRESHOLD)))           # K4
ins = instants.from_batch(fuzz.spec1_corpus(10, 300, salt=7), salt=1, p_orphan=0.02,
                          p_mismatch=0.02, p_lost=0.03)
_, _, _, wb = xm.reconstruct(xm.DeviceInstants.from_host(ins.addr, ins.bytes, ins.stream, ins.off))
xm.peaks(xm.simulate_batch(wb))                                                # K5
p = cpu_profile.batch([("mobilenet_v2", "adam", "pos0", 200, False), ("gpt2", "adamw", "pos1", 5, True)])
_, _, _, ob = xm.orchestrate(xm.DeviceProfiles.from_host(p))
xm.peaks(xm.simulate_batch(ob))                                                # K6
ts, ad, by, st, off = cpu_profile.to_instants(p)
h, _, _ = xm.estimate(xm.DeviceInstants.from_host(ad, by, st, off), torch.from_numpy(ts).cuda(),
                      p.win, p.woff)                                           # pipeline
r = np.zeros(100, xm.RUN_DTYPE)
r["m_max"] = 8 << 30
r["m_peak_est"] = np.arange(1, 101) << 26
r["oom_pred"] = r["m_peak_est"] > r["m_max"]
r["oom1"] = r["oom_pred"]
r["oom2"] = np.where(r["oom1"] == 0, 0, 2)
r["m_peak_meas1"] = 1 << 30
r["m_peak_meas2"] = 1 << 30
xm.metrics(r)                                                                  # metrics
torch.cuda.synchronize()
# raw path with the loader overlapped with the replay (> 148 x 14 traces). The
# kernels wait on each other, so a tool that serialises kernels makes the
# bounded waits give up (an XMemError, reported here) instead of hanging.
ob_ = fuzz.spec1_corpus(2300, 24, salt=9)
pb = torch.from_numpy(ob_.bytes).pin_memory().numpy()
pt = torch.from_numpy(ob_.tag.view(np.int32)).pin_memory().numpy().view(np.uint32)
try:
    xm.simulate_raw(pb, pt, ob_.off, xm.Config())                             # overlapped raw path
    print("overlapped raw path: ok, launches", xm.last_launch_count())
except xm.XMemError as e:
    print("overlapped raw path: gave up under the tool:", e)
torch.cuda.synchronize()
print("sanitize run done")
