"""N>1 on real GPUs (needs >= 2 visible; skipped on a one-GPU box): two ranks
over NCCL, each replaying its LPT shard of a config-4 slice with K2, the 64 B
results all-gathered (paper_2510_21048_b200/dist.py) -- byte-identical to one
rank replaying everything, on every rank; the summary all-reduce agrees."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch.distributed as dist
    import paper_2510_21048_b200 as xm
    from paper_2510_21048_b200.dist import gather_results, lpt_plan, reduce_summary
    from workloads import suites
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    b = suites.config4().subset(range(0, 5209, 7))
    plan = lpt_plan(b.lengths(), world)
    mine = b.subset(plan.shards[rank])
    tr = xm.load_traces(mine.bytes, mine.tag, mine.off)
    out = xm.simulate_batch(tr.to_device(dev, capacity=mine.capacity))
    full = gather_results(out, plan, rank)
    _, summ = xm.peaks(out)
    tot = reduce_summary(summ, device=dev)
    q.put((rank, full.cpu().numpy(), tot))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_gather_equals_one_rank():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (this box has %d)" % torch.cuda.device_count())
    import torch.multiprocessing as mp
    import paper_2510_21048_b200 as xm
    from workloads import suites
    b = suites.config4().subset(range(0, 5209, 7))
    tr = xm.load_traces(b.bytes, b.tag, b.off)
    ref = xm.simulate_batch(tr.to_device("cuda:0", capacity=b.capacity)).cpu().numpy()
    _, rsum = xm.peaks(xm.simulate_batch(tr.to_device("cuda:0", capacity=b.capacity)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    for rank, full, tot in got:
        assert full.tobytes() == ref.tobytes(), rank
        for k in ("n_traces", "events_done", "n_oom", "max_peak_reserved", "sum_peak_reserved"):
            assert tot[k] == rsum[k], (rank, k)
