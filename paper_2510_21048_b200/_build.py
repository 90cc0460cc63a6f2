"""In-tree build of libxmem.so for sm_100a (nvcc; no JIT cache, no torch types)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
DEBUG = bool(os.environ.get("XM_DEBUG"))
TIMING = bool(os.environ.get("XM_TIMING"))
TAG = os.environ.get("XM_BUILD_TAG", "")          # A/B tooling: a separately named variant
LIB = os.path.join(PKG, "libxmem_debug.so" if DEBUG else ("libxmem_timing.so" if TIMING else
                                                         (f"libxmem_{TAG}.so" if TAG else "libxmem.so")))
SOURCES = ["loader.cpp", "capi.cu", "replay.cu", "scan.cu", "expand.cu", "metrics.cu", "lifecycle.cu", "orchestrate.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "xmem.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    bdir = os.path.join(PKG, "build")
    os.makedirs(bdir, exist_ok=True)
    for src in SOURCES:
        obj = os.path.join(bdir, src + (".dbg.o" if DEBUG else (".tim.o" if TIMING else (f".{TAG}.o" if TAG else ".o"))))
        path = os.path.join(CSRC, src)
        if src == "replay.cu" and os.environ.get("XM_REPLAY_SRC"):   # A/B tooling
            path = os.path.abspath(os.environ["XM_REPLAY_SRC"])
        if src == "scan.cu" and os.environ.get("XM_SCAN_SRC"):       # A/B tooling
            path = os.path.abspath(os.environ["XM_SCAN_SRC"])
        if src == "lifecycle.cu" and os.environ.get("XM_LIFECYCLE_SRC"):   # A/B tooling
            path = os.path.abspath(os.environ["XM_LIFECYCLE_SRC"])
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", *(["-DXM_DEBUG"] if DEBUG else []), *(["-DXM_TRACE"] if os.environ.get("XM_TRACE") else []), *(["-DXM_TIMING"] if TIMING else []),
               *([f"-DXM_HEAP_RESERVE_DIV={os.environ['XM_HEAP_RESERVE_DIV']}"] if os.environ.get("XM_HEAP_RESERVE_DIV") else []),
               *([f"-DXM_F_INIT_DIV={os.environ['XM_F_INIT_DIV']}"] if os.environ.get("XM_F_INIT_DIV") else []),
               *([f"-DXM_ORCH_SMEM_KEYS={os.environ['XM_ORCH_SMEM_KEYS']}"] if os.environ.get("XM_ORCH_SMEM_KEYS") else []),
               *([f"-DXM_PAGE={os.environ['XM_PAGE']}"] if os.environ.get("XM_PAGE") else []),
               *([f"-DXM_K1_WARPS={os.environ['XM_K1_WARPS']}"] if os.environ.get("XM_K1_WARPS") else []),
               *([f"-DXM_MAX_NAP={os.environ['XM_MAX_NAP']}"] if os.environ.get("XM_MAX_NAP") else []),
               *([f"-DXM_K1_PER_LANE={os.environ['XM_K1_PER_LANE']}"] if os.environ.get("XM_K1_PER_LANE") else []),
               *[f"-D{k}={os.environ[k]}" for k in ("XM_K1C_PER", "XM_K1C_STAGES", "XM_K1C_CTAS_PER_SM", "XM_K1C_THREADS",
                           "XM_F_GROW_NUM", "XM_F_GROW_DEN", "XM_K1_MINB", "XM_K2_THREADS", "XM_K2_WARPS", "XM_K2_UNROLL")
                 if os.environ.get(k)],
               "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-Wall", "-I", INCLUDE, "-I", CSRC, "-c", path,
               "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    import sys
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
