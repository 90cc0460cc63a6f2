"""Multi-GPU sharding of a trace batch.

Traces are independent, so the path shards with no data-path collective:
every rank computes the same deterministic longest-processing-time (LPT) plan
from the per-trace event counts, replays only its shard, and the per-trace
64 B results are gathered once per batch with one all_gather_into_tensor
(NCCL over NVLink/NVSwitch; gloo on CPU for tests). Scaling is weak: each rank
holds a fixed share of the work.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass
from typing import List

import numpy as np


@dataclass
class ShardPlan:
    world: int
    shards: List[np.ndarray]    # global trace indices per rank (in replay order)
    events: np.ndarray          # events per rank

    def __post_init__(self):
        self._cache = {}        # per device: gather permutation and padded buffers

    @property
    def max_shard(self) -> int:
        return max((len(s) for s in self.shards), default=0)

    def perm(self, device):
        """Global trace t's row in the rank-major padded gather, as a device
        tensor built once per device (not re-uploaded every step)."""
        key = ("perm", str(device))
        if key not in self._cache:
            import torch
            M = self.max_shard
            T = sum(len(s) for s in self.shards)
            src = np.concatenate([r * M + np.arange(len(s)) for r, s in enumerate(self.shards)]) \
                if T else np.zeros(0, np.int64)
            dst = np.concatenate(self.shards) if T else np.zeros(0, np.int64)
            p = np.empty(T, np.int64)
            p[dst] = src
            self._cache[key] = torch.from_numpy(p).to(device)
        return self._cache[key]

    def buffers(self, device, width):
        """(pad [M, width], full [W*M, width]) uint8 gather buffers, reused."""
        key = ("buf", str(device), width)
        if key not in self._cache:
            import torch
            M = self.max_shard
            self._cache[key] = (torch.zeros((M, width), dtype=torch.uint8, device=device),
                                torch.empty((self.world * M, width), dtype=torch.uint8, device=device))
        return self._cache[key]


def lpt_plan(lengths: np.ndarray, world: int) -> ShardPlan:
    """Greedy LPT: traces by decreasing length, each to the least-loaded rank
    (ties -> lowest rank). Deterministic for identical inputs on every rank."""
    lengths = np.asarray(lengths, np.int64)
    order = np.argsort(-lengths, kind="stable")
    heap = [(0, r) for r in range(world)]
    heapq.heapify(heap)
    buckets: List[List[int]] = [[] for _ in range(world)]
    loads = np.zeros(world, np.int64)
    for t in order:
        load, r = heapq.heappop(heap)
        buckets[r].append(int(t))
        load += int(lengths[t])
        loads[r] = load
        heapq.heappush(heap, (load, r))
    return ShardPlan(world, [np.asarray(b, np.int64) for b in buckets], loads)


def gather_results(local, plan: ShardPlan, rank: int, group=None):
    """all_gather_into_tensor of per-rank uint8[T_r, 64] results (padded to the
    largest shard). Returns uint8[T_total, 64] in GLOBAL trace order on every
    rank (same device as `local`)."""
    import torch
    import torch.distributed as dist
    W = plan.world
    M = plan.max_shard
    width = local.shape[1] if local.dim() == 2 else 64
    # gloo (CPU tests, debugging) gathers host tensors; NCCL the device ones
    dev = "cpu" if dist.get_backend(group) == "gloo" else local.device
    pad, full = plan.buffers(dev, width)
    pad[: local.shape[0]] = local.to(dev)
    dist.all_gather_into_tensor(full, pad, group=group)
    return reorder(full, plan).to(local.device)


def reorder(full, plan: ShardPlan):
    """[W*M, 64] rank-major padded results -> [T_total, 64] in global order."""
    return full.index_select(0, plan.perm(full.device))


SUM_KEYS = ("n_traces", "events_done", "n_oom", "n_overflow", "sum_peak_reserved", "n_predicted_oom")
MAX_KEYS = ("max_peak_reserved", "max_peak_allocated")


def reduce_summary(summ: dict, device=None, group=None) -> dict:
    """Batch summary (xm_peaks' xm_summary as a dict) over all ranks: counters
    summed, peaks maxed -- two small all_reduce calls."""
    import torch
    import torch.distributed as dist
    dev = device if device is not None and dist.get_backend(group) != "gloo" else "cpu"
    s = torch.tensor([int(summ[k]) for k in SUM_KEYS], dtype=torch.int64, device=dev)
    m = torch.tensor([int(summ[k]) for k in MAX_KEYS], dtype=torch.int64, device=dev)
    dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    out = dict(summ)
    out.update({k: int(v) for k, v in zip(SUM_KEYS, s.tolist())})
    out.update({k: int(v) for k, v in zip(MAX_KEYS, m.tolist())})
    return out
