"""Per-event (allocated_blk, reserved) curve of a trace through the real torch allocator."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from workloads import suites
b = suites.config2().subset([31])
by, tg = b.trace(0)
os.environ.pop("PYTORCH_CUDA_ALLOC_CONF", None)
dev = torch.device("cuda", 0)
torch.cuda.empty_cache()
live = {}
cur = np.zeros((len(by), 3), np.int64)
addr = np.zeros(len(by), np.int64)
for i in range(len(by)):
    v = int(by[i]); bid = int(tg[i]) & ((1 << 28) - 1)
    if v > 0:
        live[bid] = torch.empty(v, dtype=torch.uint8, device=dev)
        addr[i] = live[bid].data_ptr()
    else:
        del live[bid]
    cur[i, 0] = torch.cuda.memory_allocated(0)
    cur[i, 1] = torch.cuda.memory_reserved(0)
np.savez("gpurun_out/torch_curve.npz", curve=cur, addr=addr)
print("done", cur[:, 1].max())
