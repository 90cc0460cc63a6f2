"""Per-trace replay start/end inside xm_simulate_raw (XM_TIMING build: the
replay records globaltimer per trace in its scratch): when did the longest
traces start, when did the last ones end."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("XM_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             "paper_2510_21048_b200", "libxmem_timing.so"))
import numpy as np, torch
import paper_2510_21048_b200 as xm
from workloads import suites
b = suites.config4()
pin_b = torch.from_numpy(b.bytes).pin_memory().numpy()
pin_t = torch.from_numpy(b.tag.view(np.int32)).pin_memory().numpy().view(np.uint32)
_, ws = xm.simulate_raw(pin_b, pin_t, b.off, xm.Config(), capacity=b.capacity)
_, ws = xm.simulate_raw(pin_b, pin_t, b.off, xm.Config(), capacity=b.capacity, workspace=ws)
T = b.n_traces
raw = ws.cpu().numpy()
# the timing array is the last T*16 bytes of the replay scratch, which ends the workspace
need = int(xm.lib().xm_raw_ws_bytes(b.off.ctypes.data_as(__import__("ctypes").c_void_p), T,
                                    __import__("ctypes").byref(xm.Config().c())))
# the timing array ([T][2] u64) ends the replay scratch, which ends the
# workspace up to <= 255 bytes of alignment: find the 8-byte shift at which
# every entry reads as a globaltimer value
tail = raw[max(0, need - 16 * T - 256): need]
tm = None
for sh in range(0, 257, 8):
    seg = tail[len(tail) - sh - 16 * T: len(tail) - sh] if sh else tail[len(tail) - 16 * T:]
    v = seg.view(np.uint64).reshape(T, 2)
    if (v[:, 0] > 10**18).all() and (v[:, 1] >= v[:, 0]).all():
        tm = v.astype(np.float64)
        break
assert tm is not None, "timing array not found"
ok = tm[:, 0] > 0
t0 = tm[ok, 0].min()
st = (tm[:, 0] - t0) / 1e6
en = (tm[:, 1] - t0) / 1e6
L = b.lengths()
o = np.argsort(-L)
print("traces timed", ok.sum(), "of", T, " makespan %.2f ms" % en[ok].max())
for k in [0, 1, 10, 100, 379, 1000, 2072, 3000, 5208]:
    t = o[k]
    print(f"LPT rank {k:5d} len {L[t]:6d} start {st[t]:7.3f} end {en[t]:7.3f} ms")
late = np.argsort(-en)[:8]
for t in late:
    print(f"late: len {L[t]:6d} start {st[t]:7.3f} end {en[t]:7.3f} ns/ev {(en[t]-st[t])*1e6/max(L[t],1):.0f}")
