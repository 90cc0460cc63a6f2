"""Multi-rank host logic on CPU (gloo, world_size 2): identical LPT plans on
every rank, and the gathered results equal a single-rank run in global order."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_21048_b200.dist import gather_results, lpt_plan, reduce_summary, reorder


def test_lpt_plan_properties():
    rng = np.random.default_rng(0)
    L = rng.integers(500, 25000, 5209)
    for W in (1, 2, 4, 8):
        p = lpt_plan(L, W)
        allidx = np.sort(np.concatenate(p.shards))
        assert (allidx == np.arange(len(L))).all()
        assert p.events.sum() == L.sum()
        # LPT bound: makespan <= 4/3 OPT; OPT >= mean and >= max
        assert p.events.max() <= (4 / 3) * max(L.sum() / W, L.max()) + 1
        q = lpt_plan(L, W)
        assert all((a == b).all() for a, b in zip(p.shards, q.shards))


def test_reorder_roundtrip():
    L = np.array([5, 1, 9, 3, 7, 2, 8])
    p = lpt_plan(L, 3)
    M = p.max_shard
    full = torch.zeros((3 * M, 64), dtype=torch.uint8)
    for r, s in enumerate(p.shards):
        for k, t in enumerate(s):
            full[r * M + k, 0] = int(t) + 1
    out = reorder(full, p)
    assert out[:, 0].tolist() == [t + 1 for t in range(len(L))]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, lengths, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = lpt_plan(lengths, world)
    mine = plan.shards[rank]
    # fake per-trace result: record bytes derived from the global index
    local = torch.zeros((len(mine), 64), dtype=torch.uint8)
    for k, t in enumerate(mine):
        local[k, :8] = torch.tensor(list(int(t * 7 + 3).to_bytes(8, "little")), dtype=torch.uint8)
    out = gather_results(local, plan, rank)
    q.put((rank, out.numpy().copy(), [s.tolist() for s in plan.shards]))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_gloo_world2():
    lengths = np.random.default_rng(1).integers(10, 1000, 37)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, lengths, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    (r0, o0, s0), (r1, o1, s1) = sorted(res, key=lambda x: x[0])
    assert s0 == s1                                   # identical plans on both ranks
    assert (o0 == o1).all()
    vals = o0[:, :8].copy().view(np.uint64).ravel()
    assert vals.tolist() == [t * 7 + 3 for t in range(len(lengths))]


def _oracle_worker(rank, world, port, q):
    """Each rank replays its LPT shard of real traces (with the oracle, as a
    stand-in for its GPU) and the per-trace records are all-gathered."""
    import oracle
    from workloads import fuzz, mc5
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = np.arange(0, 3000, 97)                      # config-5 traces (global indices)
    lengths = mc5.lengths(mc5.describe(idx))
    plan = lpt_plan(lengths, world)
    mine = plan.shards[rank]
    b = mc5.batch(idx[mine])
    o = oracle.simulate_batch(b)
    rec = np.zeros((len(mine), 8), np.uint64)
    for c, f in enumerate(["peak_allocated", "peak_allocated_blk", "peak_reserved", "final_reserved",
                           "events_done", "status", "n_seg_alloc", "n_seg_release"]):
        rec[:, c] = o[f]
    local = torch.from_numpy(rec.view(np.uint8).reshape(len(mine), 64).copy())
    out = gather_results(local, plan, rank)
    summ = {"n_traces": len(mine), "events_done": int(o["events_done"].sum()),
            "n_oom": int((o["status"] == 1).sum()), "n_overflow": 0,
            "sum_peak_reserved": int(o["peak_reserved"].sum()), "n_predicted_oom": 0,
            "max_peak_reserved": int(o["peak_reserved"].max()),
            "max_peak_allocated": int(o["peak_allocated"].max())}
    q.put((rank, out.numpy().copy(), reduce_summary(summ)))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_replay_gloo_equals_single_rank():
    import oracle
    from workloads import mc5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_oracle_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    (_, o0, s0), (_, o1, s1) = sorted(res, key=lambda x: x[0])
    assert (o0 == o1).all() and s0 == s1
    idx = np.arange(0, 3000, 97)
    whole = oracle.simulate_batch(mc5.batch(idx))
    assert s0["n_traces"] == len(idx) and s0["events_done"] == int(whole["events_done"].sum())
    assert s0["n_oom"] == int((whole["status"] == 1).sum())
    assert s0["max_peak_reserved"] == int(whole["peak_reserved"].max())
    got = o0.view(np.uint64).reshape(len(idx), 8)
    for c, f in enumerate(["peak_allocated", "peak_allocated_blk", "peak_reserved", "final_reserved",
                           "events_done", "status", "n_seg_alloc", "n_seg_release"]):
        assert (got[:, c] == whole[f]).all(), f
