import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import ctypes
import paper_2510_21048_b200 as xm
from paper_2510_21048_b200 import _build
if os.environ.get("XM_DEBUG"):
    xm._lib = None
    _build.LIB = os.path.join(_build.PKG, "libxmem_debug.so")
from workloads import concat, hand, fuzz
import oracle
from gpu_util import gpu_run, oracle_run, assert_parity
named = hand.all_named()
named["frag"] = fuzz.fragmentation_stress()
named["frag2"] = fuzz.fragmentation_stress(8192, 1024, "frag2")
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which == "all":
    b = concat(list(named.values()))
else:
    b = concat([named[k] for k in which.split(",")])
cfg = xm.Config(smem_per_warp=int(os.environ.get("SPW", "0")), warps_per_cta=int(os.environ.get("WPC", "0")))
h, s = gpu_run(b, cfg)
o = oracle_run(b)
assert_parity(b, h, o)
print("OK", b.n_traces)
