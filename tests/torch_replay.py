"""Replay traces through the REAL PyTorch CUDACachingAllocator (run as a
subprocess on a GPU box) and record what it did.

The paper's Simulator "follows the PyTorch Official implementation" (PAPER.md:257
footnote); this is the external pin SURVEY.md §4.3 plans: alloc = torch.empty of
the request on the event's stream, free = drop the tensor (no record_stream), a
finite capacity = torch.cuda.set_per_process_memory_fraction. Used only by
tests/test_torch_allocator_pin.py.

usage: torch_replay.py IN.npz OUT.npz [ALLOC_CONF]   (IN: bytes, tag, off, capacity)
ALLOC_CONF: optional PYTORCH_CUDA_ALLOC_CONF for the replay (allocator variants).
OUT: stats (JSON string, one dict per trace), and per event: allocated bytes,
reserved bytes (+ with XM_PIN_SEGMENTS=1 the segments obtained so far) and the
returned device pointer (0 for frees).
"""
import json
import os
import sys

import numpy as np


def replay_one(torch, by, tg, cap, curve, ptr):
    dev = torch.device("cuda", 0)
    total = torch.cuda.mem_get_info(0)[1]            # cudaMemGetInfo, as torch's setMemoryFraction
    frac = min(1.0, cap / total)
    torch.cuda.set_per_process_memory_fraction(frac, 0)
    allowed = int(frac * float(total))               # static_cast<size_t>(fraction * double(total))
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats(0)
    base = torch.cuda.memory_stats(0)
    seg0 = base.get("segment.all.allocated", 0)
    streams = {0: torch.cuda.current_stream(0)}
    live = {}
    fail = -1
    for i in range(len(by)):
        b = int(by[i])
        bid = int(tg[i]) & ((1 << 28) - 1)
        st = int(tg[i]) >> 28
        if b > 0:
            if st not in streams:
                streams[st] = torch.cuda.Stream(0)
            try:
                with torch.cuda.stream(streams[st]):
                    x = torch.empty(b, dtype=torch.uint8, device=dev)
            except torch.OutOfMemoryError:
                fail = i
                break
            live[bid] = x
            ptr[i] = x.data_ptr()
            del x                     # the only reference must be live[bid]
        else:
            del live[bid]
        curve[i, 0] = torch.cuda.memory_allocated(0)
        curve[i, 1] = torch.cuda.memory_reserved(0)
        if curve.shape[1] > 2:        # segments obtained so far (new segment at i: it grew)
            curve[i, 2] = torch.cuda.memory_stats(0)["segment.all.allocated"] - seg0
    s = torch.cuda.memory_stats(0)
    out = {
        "peak_allocated_blk": s["allocated_bytes.all.peak"],
        "peak_reserved": s["reserved_bytes.all.peak"],
        "final_reserved": s["reserved_bytes.all.current"],
        "n_seg_alloc": s["segment.all.allocated"] - base.get("segment.all.allocated", 0),
        "n_seg_release": s["segment.all.freed"] - base.get("segment.all.freed", 0),
        "max_live_segments": s["segment.all.peak"],
        "fail_idx": fail,
        "num_ooms": s.get("num_ooms", 0) - base.get("num_ooms", 0),
        "allowed": allowed,
    }
    live.clear()
    return out


def main(inp, outp, conf=""):
    os.environ.pop("PYTORCH_CUDA_ALLOC_CONF", None)
    if conf:
        os.environ["PYTORCH_CUDA_ALLOC_CONF"] = conf
    import torch
    torch.cuda.init()
    d = np.load(inp)
    off, cap = d["off"], d["capacity"]
    E = int(off[-1])
    curve = np.zeros((E, 3 if os.environ.get("XM_PIN_SEGMENTS") else 2), np.int64)
    ptr = np.zeros(E, np.int64)
    res = []
    for t in range(len(off) - 1):
        a, b = int(off[t]), int(off[t + 1])
        res.append(replay_one(torch, d["bytes"][a:b], d["tag"][a:b], int(cap[t]),
                              curve[a:b], ptr[a:b]))
    np.savez(outp, stats=json.dumps(res), curve=curve, ptr=ptr)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
