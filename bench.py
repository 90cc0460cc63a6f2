#!/usr/bin/env python
"""Benchmark: batched caching-allocator trace replay (xMem's Simulator hot path).

One "step" = one pass of the whole hot path over
one batch: every trace of the workload replayed through xm_simulate_batch
(K2) with inputs resident in HBM, plus (N>1) the NCCL all_gather of the
per-trace results. Metric (BASELINE.json): allocator-trace events replayed per
second, whole job, with bit-exact peaks vs the CPU oracle (checked here too).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

N=1 workload: BASELINE configs[3], the 25-model suite x 5209 runs (the
single-GPU config the metric is quoted on). N>1: weak scaling -- the global
pool holds N x 5209 traces (config 4 + further Monte Carlo draws, configs[4]),
LPT-sharded so each GPU replays ~one config-4-sized shard.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "allocator-trace events replayed/s (1/2/4/8 B200), bit-exact peaks vs CPU oracle"
UNIT = "events/s"
L2_BYTES = 126 * 1024 * 1024
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--cfg5-traces", type=int, default=1_000_000,
                    help="config 5: total Monte Carlo traces (sharded over the GPUs)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-k1", action="store_true",
                    help="skip the K1 measurement (launch lists of the step alone)")
    ap.add_argument("--smem-per-warp", type=int, default=0)
    ap.add_argument("--warps-per-cta", type=int, default=0)
    ap.add_argument("--json-out", default="")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------- workload
def workload(name: str, world: int, rank: int):
    """Returns (batch for this rank, plan or None, description dict, total events, total traces)."""
    from workloads import suites
    if name != "cfg4":
        b = suites.CONFIGS[name]()
        desc = {"cfg1": "configs[0] 3-layer MLP, 1 iteration, batch 32",
                "cfg2": "configs[1] ResNet-50 sweep b=8..256 (32 traces)",
                "cfg3": "configs[2] BERT-base/GPT-2 AdamW, 3 streams (44 traces)"}[name]
        return b, None, desc, b.n_events, b.n_traces
    from paper_2510_21048_b200.dist import lpt_plan
    n = suites.N_CFG4 * world
    if world == 1:
        b = suites.config4()
        return b, None, "configs[3] 25-model suite x 5209 runs (3903 ANOVA + 1306 MC)", \
            b.n_events, b.n_traces
    lengths = suites.pool_lengths(n)
    plan = lpt_plan(lengths, world)
    b = suites.pool_batch(plan.shards[rank])
    desc = (f"configs[3]+[4]: {n} traces = config-4 suite + {n - suites.N_CFG4} Monte Carlo "
            f"draws, LPT-sharded over {world} GPUs")
    return b, plan, desc, int(lengths.sum()), n


# ---------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50",
                                       "-i", str(index)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.15)
        self.p.terminate()
        try:
            self.p.wait(5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    rows.append((float(parts[0]), float(parts[1]), float(parts[3]), parts[5:9]))
                except ValueError:
                    continue
        os.unlink(self.f.name)
        if not rows:
            return None
        load = [r for r in rows if r[2] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in load for n, v in zip(names, r[3]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in load])),
                "sm_max_mhz": float(max(r[1] for r in rows)),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(load)}


def peaks_json():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel="k_replay"):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        k = d["kernels"][kernel]
        return k["dram_bytes_per_launch"], k.get("source", p)
    except Exception:
        return None, None


def peaks_clock():
    """The SM clock MEASURED_PEAKS.json records (when no live clock sample)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("sm_max_mhz") or 0) or None
    except Exception:
        return None


def ncu_issue(kernel="k_replay", kernel_ms=None, sm_mhz=None, events=None):
    """Warp-issue efficiency (smsp__issue_active %) and warp-instructions per
    launch from the committed ncu summary (the north_star's second measure),
    plus the issue roofline of this run: frac = warp-instructions / (SMs x 4
    schedulers x SM clock x the live kernel time), one warp-instruction per
    scheduler per cycle being the ceiling."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            k = json.load(f)["kernels"][kernel]
        r = {"issue_active_pct": k["issue_active_pct"],
             "warp_instructions_per_launch": k["warp_instructions"],
             "achieved_occupancy_pct": k["achieved_occupancy_pct"],
             "source": "profiles/ncu_summary.json (" + k.get("source", "") + ")"}
        if kernel_ms and sm_mhz:
            import torch
            sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            cap = sms * 4 * sm_mhz * 1e6 * kernel_ms / 1e3
            r.update({"frac": k["warp_instructions"] / cap, "sms": sms, "sm_mhz": sm_mhz,
                      "ceiling_warp_instructions": cap})
            if events:
                r["warp_instructions_per_event"] = k["warp_instructions"] / events
        return r
    except Exception:
        return None


# ---------------------------------------------------------------- cpu oracle
def _oracle_pool():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_pool
    return oracle_pool


def oracle_rate(batch, passes=1):
    """The oracle as it stands (oracle/xmo.c) on every host core: forked workers
    inherit the batch (nothing pickled but chunk numbers) and time only the
    simulate call; the rate divides by the busiest worker's simulate time
    (SURVEY.md §8(d) "timing only simulate"). Returns (rate, detail, results)."""
    op = _oracle_pool()
    with op.Pool(batch) as pool:
        best = None
        for _ in range(passes):
            res, wall, busiest, total = pool.run()
            if best is None or busiest < best[1]:
                best = (wall, busiest, total)
        cores = pool.workers
    wall, busiest, total = best
    ev = int(res["events_done"].sum())
    return ev / busiest, {"cores": cores, "wall_s": wall, "busiest_worker_simulate_s": busiest,
                          "simulate_s_all_workers": total, "events": ev,
                          "wall_value": ev / wall, "cpu_model": op.cpu_model()}, res


def single_core_rate(batch, budget_events=4_000_000):
    """The oracle on ONE host core (SURVEY.md §8(d) oracle timing (i)), on every
    k-th trace up to ~budget_events."""
    import oracle
    k = max(1, int(np.ceil(batch.n_events / budget_events)))
    sub = batch.subset(range(0, batch.n_traces, k))
    t0 = time.perf_counter()
    r = oracle.simulate_batch(sub)
    dt = time.perf_counter() - t0
    ev = int(r["events_done"].sum())
    return {"value": ev / dt, "unit": UNIT, "cores": 1,
            "sample": f"every {k}th trace: {sub.n_traces} traces, {ev} events, {dt:.2f} s"}


def bounded_sample(batch, budget_events=60_000_000):
    """Whole workload when it is small enough, else every k-th trace."""
    if batch.n_events <= budget_events:
        return batch, f"all {batch.n_traces} traces ({batch.n_events} events)"
    k = int(np.ceil(batch.n_events / budget_events))
    idx = list(range(0, batch.n_traces, k))
    sub = batch.subset(idx)
    return sub, f"every {k}th trace: {sub.n_traces} traces ({sub.n_events} events)"


# ---------------------------------------------------------------- reference arm
def run_reference(args, world, rank):
    if rank != 0:
        return 0
    if args.workload == "cfg5":
        from workloads import mc5
        n = args.cfg5_traces
        total_tr = n
        total_ev = int(mc5.lengths(mc5.describe(np.arange(n))).sum())
        k = max(1, int(np.ceil(total_ev / 25_000_000)))
        b = mc5.batch(np.arange(0, n, k))
        desc = f"configs[4] Monte Carlo, {n} traces (every {k}th trace replayed by the oracle)"
        plan = None
    else:
        b, plan, desc, total_ev, total_tr = workload(args.workload, 1 if world == 1 else world, 0)
    if plan is not None:   # the whole pool, not rank 0's shard
        from workloads import suites
        b = suites.pool_batch(range(total_tr))
    sample, sdesc = bounded_sample(b, 30_000_000)
    op = _oracle_pool()
    times = []
    busiest = []
    ev = 0
    with op.Pool(sample) as pool:           # forked once; every step re-runs the oracle
        cores = pool.workers
        for _ in range(args.warmup):
            pool.run()
        for _ in range(args.steps):
            r, wall, busy, _ = pool.run()
            times.append(wall)
            busiest.append(busy)
            ev = int(r["events_done"].sum())
    ms = 1e3 * float(np.mean(times))
    value = ev / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if args.workload == "cfg5" else "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": desc, "sample": sdesc, "n_traces": total_tr,
                       "n_events": total_ev},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sdesc, "cpu_model": op.cpu_model(),
                             "timing": "wall time of one pass of forked workers (inputs inherited "
                                       "at fork, results returned); busiest worker's simulate-only "
                                       "rate in simulate_only_value",
                             "simulate_only_value": ev / float(np.mean(busiest))},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
def _device(local):
    """cuda:LOCAL_RANK. XM_BENCH_DEVICE=k pins every rank to GPU k -- a
    debugging aid only, to run the N>1 code path on a one-GPU box (with
    XM_BENCH_BACKEND=gloo; NCCL refuses two ranks on one GPU)."""
    import torch
    k = int(os.environ.get("XM_BENCH_DEVICE", local))
    torch.cuda.set_device(k)
    return torch.device("cuda", k)


def _cdev(dev):
    """Device of the small all-reduce tensors: host memory under gloo."""
    import torch.distributed as dist
    return "cpu" if dist.is_initialized() and dist.get_backend() == "gloo" else dev


def _init_dist(dev):
    import torch.distributed as dist
    backend = os.environ.get("XM_BENCH_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
def relaunch(args) -> int:
    """--gpus N > 1 without a launcher: run this same command under
    torch.distributed.run, one rank per GPU, rendezvous on 127.0.0.1."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank "
                         f"per GPU (or omit the launcher and let bench.py start them)")
    if world > 1 and os.environ.get("XM_BENCH_BACKEND", "nccl") == "nccl":
        # keep NCCL's communicator-init log (rank count per communicator)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        return run_reference(args, world, rank)
    if args.workload == "cfg5":
        return main_cfg5(args, world, rank, local)

    import torch
    import torch.distributed as dist
    import paper_2510_21048_b200 as xm
    from paper_2510_21048_b200.dist import gather_results

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: CUDA device required (no CPU fallback)")
    dev = _device(local)
    if world > 1:
        _init_dist(dev)

    batch, plan, desc, total_ev, total_tr = workload(args.workload, world, rank)
    tr = xm.load_traces(batch.bytes, batch.tag, batch.off)
    has_cap = bool((batch.capacity != xm.UNLIMITED).any())
    cap = batch.capacity if has_cap else None
    db = tr.to_device(dev, capacity=cap)
    cfg = xm.Config(smem_per_warp=args.smem_per_warp, warps_per_cta=args.warps_per_cta)
    stream = torch.cuda.current_stream(dev)
    out = torch.empty((batch.n_traces, 64), dtype=torch.uint8, device=dev)
    in_bytes = 12 * batch.n_events + 24 * batch.n_traces
    flush = in_bytes < 2 * L2_BYTES
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None

    def step():
        r = xm.simulate_batch(db, cfg, stream, out=out)
        if world > 1:
            gather_results(r, plan, rank)
        return r

    sampler = ClockSampler(local) if rank == 0 or True else None
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    launches_per_step = xm.last_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t_all0 = torch.cuda.Event(enable_timing=True)
    t_all1 = torch.cuda.Event(enable_timing=True)
    t_all0.record(stream)
    for k in range(args.steps):
        if flush:
            flush_buf.fill_(k & 0xFF)
        evs[k][0].record(stream)
        step()
        evs[k][1].record(stream)
    t_all1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.sum(step_ms)) / args.steps if flush else t_all0.elapsed_time(t_all1) / args.steps
    # kernel-only durations (xm_simulate_batch, no gather) for the roofline
    kevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    for k in range(args.steps):
        kevs[k][0].record(stream)
        xm.simulate_batch(db, cfg, stream, out=out)
        kevs[k][1].record(stream)
    torch.cuda.synchronize()
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in kevs]))
    if world > 1:
        t = torch.tensor([ms, kern_ms], dtype=torch.float64, device=_cdev(dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kern_ms = float(t[0]), float(t[1])

    # results of this rank (for parity); batch summary over all ranks
    h, summ = xm.peaks(out)
    if world > 1:
        from paper_2510_21048_b200.dist import reduce_summary
        summ = reduce_summary(summ, device=dev)
    local_done = int(h["events_done"].astype(np.int64).sum())
    done = local_done
    if world > 1:
        t = torch.tensor([local_done], dtype=torch.int64, device=_cdev(dev))
        dist.all_reduce(t)
        done = int(t[0])
    value = done / (ms / 1e3)

    # ---- e2e through the host-buffer C-ABI entry point (H2D + replay + D2H)
    e2e = None
    if not args.no_e2e:
        ws = None
        capn = np.ascontiguousarray(batch.capacity, np.uint64) if has_cap else None

        def e2e_ms(mode, from_raw=False):
            """Mean wall time of xm_simulate_host with event input `mode`
            (XM_HOST_INPUT, capi.cu; None = the library default). from_raw:
            every step starts from the caller's raw arrays, i.e. includes
            xm_load_traces (validation S:231/S:249/S:258, dense renumbering,
            LPT order, page-locked packing; SURVEY.md §8(d) end-to-end)."""
            nonlocal ws
            old_mode = os.environ.pop("XM_HOST_INPUT", None)
            if mode:
                os.environ["XM_HOST_INPUT"] = mode

            def one():
                t_ = xm.load_traces(batch.bytes, batch.tag, batch.off) if from_raw else tr
                return xm.simulate_host(t_, cfg, capacity=capn, workspace=ws)
            try:
                for _ in range(2):
                    _, ws = one()
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                for _ in range(args.steps):
                    hh, ws = one()
                dt = (time.perf_counter() - t0) / args.steps
            finally:
                os.environ.pop("XM_HOST_INPUT", None)
                if old_mode is not None:
                    os.environ["XM_HOST_INPUT"] = old_mode
            if world > 1:
                t = torch.tensor([dt], dtype=torch.float64, device=_cdev(dev))
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = float(t[0])
            return dt, hh

        # the headline: xm_simulate_raw on the caller's raw arrays in page-locked
        # host memory (pinned once, as a user's input buffers would be): the
        # device validates, renumbers and replays (k_load overlapped with k_replay) every step
        pin_b = torch.from_numpy(np.ascontiguousarray(batch.bytes)).pin_memory().numpy()
        pin_t = torch.from_numpy(np.ascontiguousarray(batch.tag).view(np.int32)).pin_memory() \
            .numpy().view(np.uint32)
        rws = None
        for _ in range(2):
            _, rws = xm.simulate_raw(pin_b, pin_t, batch.off, cfg, capacity=capn, workspace=rws)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            h_dev_raw, rws = xm.simulate_raw(pin_b, pin_t, batch.off, cfg, capacity=capn,
                                             workspace=rws)
        dt_dev_raw = (time.perf_counter() - t0) / args.steps
        if world > 1:
            t = torch.tensor([dt_dev_raw], dtype=torch.float64, device=_cdev(dev))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt_dev_raw = float(t[0])
        del rws
        dt_raw, h_raw = e2e_ms(None, from_raw=True)
        dt, h_e2e = e2e_ms(None)
        dt_stream, h_stream = e2e_ms("stream")
        ev_bytes = 8 if tr.packed is not None else 12        # packed or bytes + tag
        h2d = ev_bytes * batch.n_events + 8 * (batch.n_traces + 1) \
            + 8 * batch.n_traces + (8 * batch.n_traces if has_cap else 0)
        direct = tr.packed is not None and not os.environ.get("XM_NO_STREAM") \
            and os.environ.get("XM_HOST_INPUT", "direct") == "direct"
        h2d_raw = 12 * batch.n_events + 8 * (batch.n_traces + 1) + 4 * batch.n_traces \
            + (8 * batch.n_traces if has_cap else 0)
        e2e = {"value": done / dt_dev_raw, "unit": UNIT, "h2d_bytes_per_step": int(h2d_raw),
               "d2h_bytes_per_step": int(128 * batch.n_traces), "ms_per_step": dt_dev_raw * 1e3,
               "api": "xm_simulate_raw: the caller's raw arrays (page-locked host memory) "
                      "copied to the device in 48 chunks of whole traces on a copy stream; "
                      "the device loader (k_load, keyed by raw block id: validation "
                      "S:231/S:249/S:258, dense ids, LPT-stored wire arrays) on 16 SMs, "
                      "longest first among the traces whose chunk has landed, appending each "
                      "finished trace to a completion queue; k_replay on the other SMs from "
                      "the start, popping that queue, then on the loader's SMs too -> results "
                      "+ loader verdicts to the host, every step",
               "host_loader": {"value": done / dt_raw, "ms_per_step": dt_raw * 1e3,
                               "api": "xm_load_traces (host validation, dense ids, page-locked "
                                      "packing) + xm_simulate_host, every step",
                               "h2d_bytes_per_step": int(h2d)},
               "pinned_handle": {"value": done / dt, "ms_per_step": dt * 1e3},
               "pinned_handle_api": "xm_simulate_host on an already loaded handle (pinned host traces -> device -> host results; "
                      + ("events read by the replaying warps straight from the page-locked "
                         "host array over PCIe, no staging copy; " if direct else
                         "upload streamed in longest-first chunks overlapping the replay; ")
                      + ("8-byte packed events)" if tr.packed is not None else "12-byte events)"),
               "stream_copy_ms_per_step": dt_stream * 1e3,
               "results_equal_device_path": bool((h_e2e == h).all() and (h_stream == h).all()
                                                 and (h_raw == h).all() and (h_dev_raw == h).all())}
    clocks = sampler.stop() if sampler else None

    # ---- roofline of the dominant kernel (k_replay): algorithmic bytes / launch time
    # (12 B per replayed event read once, 24 B/trace descriptors, 64 B/trace out)
    alg = 12 * local_done + 24 * batch.n_traces + 64 * batch.n_traces
    peak, peak_src = peaks_json()
    achieved = alg / (kern_ms / 1e3) / 1e9
    traffic, tsrc = ncu_traffic()
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "kernel": "k_replay",
            "alg_bytes_per_launch": alg, "kernel_ms": kern_ms, "peak_source": peak_src,
            "traffic_source": tsrc,
            # (the committed ncu capture is of the N=1 config-4 batch: the
            # issue fraction is computed only for that launch)
            "issue": (ncu_issue("k_replay", kern_ms,
                                (clocks or {}).get("sm_mhz") or peaks_clock(), local_done)
                      if world == 1 else ncu_issue()),
            "note": "K2 is a serial integer state machine per trace (issue/latency-bound); "
                    "HBM fraction reported as the north_star asks, warp-issue efficiency "
                    "from ncu in 'issue'"}

    # ---- K1 (XM_ALLOCATED_ONLY: segmented prefix-scan/max), the HBM-bound kernel,
    # timed on the same resident events (capacities dropped: the mode needs none)
    k1 = None
    try:
        if args.no_k1:
            raise RuntimeError("skipped (--no-k1)")
        db1 = xm.DeviceBatch(db.bytes, db.tag, db.off, db.n_ids, db.order, None, db.n_traces,
                             db.n_events, db.max_ids, db.max_events)
        cfg1 = xm.Config(mode=1)
        out1 = torch.empty_like(out)
        for _ in range(3):
            xm.simulate_batch(db1, cfg1, stream, out=out1)
        # K1's launch (~50 us) is shorter than the host's call overhead, so a
        # launch timed alone between two events also times the host gap before
        # it: each sample times `reps` launches queued back to back (the
        # inputs, 233+ MB, exceed L2, so no launch reads the previous one's
        # data from cache) and reports the mean launch duration
        ks = []
        reps = 20
        for _ in range(max(5, args.steps)):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if flush:
                flush_buf.fill_(1)
            a0.record(stream)
            for _r in range(reps):
                xm.simulate_batch(db1, cfg1, stream, out=out1)
            a1.record(stream)
            torch.cuda.synchronize()
            ks.append(a0.elapsed_time(a1) / reps)
        k1_ms = float(np.median(ks))
        k1_alg = 8 * batch.n_events + 8 * (batch.n_traces + 1) + 64 * batch.n_traces
        k1_ach = k1_alg / (k1_ms / 1e3) / 1e9
        k1 = {"kernels": {"c": "k_scan_chunks (K1c, TMA)", "t": "k_scan_trace (K1t)",
                          "f": "k_row_map + k_scan_tiles + k_scan_combine"}[
                              (os.environ.get("XM_K1") or
                               ("t" if batch.lengths().max(initial=0) <= 65536 else "c"))[0]],
              "ms": k1_ms,
              "timing": f"mean of {reps} back-to-back launches per sample, median of samples",
              "events_per_s": batch.n_events / (k1_ms / 1e3), "bound": "hbm",
              "achieved": k1_ach, "peak": peak, "unit": "GB/s", "frac": k1_ach / peak,
              "alg_bytes_per_launch": k1_alg}
    except Exception as e:  # reported, never fatal for the main metric
        k1 = {"error": str(e)}

    # ---- cpu baseline (oracle) + parity of every trace of this rank (rank 0, N=1)
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample, sdesc = bounded_sample(batch)
        rate, det, o = oracle_rate(sample)
        cpu = {"value": rate, "unit": UNIT, "cores": det["cores"], "kind": "oracle",
               "sample": sdesc + f"; busiest of {det['cores']} forked workers simulated for "
                                 f"{det['busiest_worker_simulate_s']:.2f} s",
               "cpu_model": det["cpu_model"], "wall_value": det["wall_value"],
               "single_core": single_core_rate(batch)}
        if not args.no_parity and sample.n_traces == batch.n_traces:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from gpu_util import COMPARE
            mism = 0
            for f in COMPARE:
                exp = o[f].astype(np.uint64)
                if f == "n_free_blocks_end":
                    exp = np.minimum(exp, 65535)
                mism += int((h[f].astype(np.uint64) != exp).sum())
            parity = {"traces": batch.n_traces, "fields": len(COMPARE),
                      "mismatched_values": mism}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic",
            "config": {"workload": desc, "n_traces": total_tr, "n_events": total_ev,
                       "events_done": done, "traces_per_s": total_tr / (ms / 1e3),
                       "l2": ("flushed (256 MiB write) between steps" if flush else
                              f"inputs larger than L2 ({in_bytes / 2**20:.0f} MiB/GPU > 126 MiB)"),
                       "parallelism": f"dp{world} (trace-sharded)",
                       "smem_per_warp": args.smem_per_warp or "auto",
                       "n_oom": summ["n_oom"], "n_overflow": summ["n_overflow"]},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roof, "roofline_k1_allocated_only": k1, "cpu_baseline": cpu,
            "e2e": e2e, "clocks": clocks, "parity": parity}
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(s + "\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------- config 5
def main_cfg5(args, world, rank, local):
    """configs[4]: N Monte Carlo traces (default 1M) generated ON
    THE DEVICE by K4 from ~200 templates (only descriptors cross PCIe), LPT-
    sharded over the GPUs (strong scaling: the total is fixed), replayed by K2,
    per-trace results all-gathered (N>1). Timed step = replay (+ gather)."""
    import torch
    import torch.distributed as dist
    import paper_2510_21048_b200 as xm
    from paper_2510_21048_b200.dist import gather_results, lpt_plan
    from workloads import mc5

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: CUDA device required (no CPU fallback)")
    dev = _device(local)
    if world > 1:
        _init_dist(dev)
    n = args.cfg5_traces
    d_all = mc5.describe(np.arange(n))
    L = mc5.lengths(d_all)
    plan = lpt_plan(L, world) if world > 1 else None
    mine = plan.shards[rank] if plan else np.arange(n)
    d = {k: v[mine] for k, v in d_all.items()}
    pool = xm.Templates(*mc5.template_pool(), device=dev)
    stream = torch.cuda.current_stream(dev)
    # K4 (generation, not timed in the step; its kernel timed separately on a
    # re-expansion into the same buffers: one launch)
    db = xm.expand_templates(pool, d["tpl"], d["b"], d["seed"], mc5.SWAP_THRESHOLD,
                             capacity=d["capacity"], stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    xm.expand_again(pool, db, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    k4_ms = e0.elapsed_time(e1)
    cfg = xm.Config(smem_per_warp=args.smem_per_warp, warps_per_cta=args.warps_per_cta)
    out = torch.empty((len(mine), 64), dtype=torch.uint8, device=dev)

    def step():
        r = xm.simulate_batch(db, cfg, stream, out=out)
        if world > 1:
            gather_results(r, plan, rank)
        return r

    sampler = ClockSampler(local)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    launches = xm.last_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1) / args.steps
    kt0, kt1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kt0.record(stream)
    for _ in range(args.steps):
        xm.simulate_batch(db, cfg, stream, out=out)
    kt1.record(stream)
    torch.cuda.synchronize()
    kern_ms = kt0.elapsed_time(kt1) / args.steps
    h, summ = xm.peaks(out)
    if world > 1:
        from paper_2510_21048_b200.dist import reduce_summary
        summ = reduce_summary(summ, device=dev)
    local_done = int(h["events_done"].astype(np.int64).sum())
    vals = torch.tensor([ms, kern_ms, k4_ms, float(local_done)], dtype=torch.float64, device=_cdev(dev))
    if world > 1:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm)
        ms, kern_ms, k4_ms, done = float(mx[0]), float(mx[1]), float(mx[2]), int(sm[3])
    else:
        done = local_done
    value = done / (ms / 1e3)

    # e2e through the public API: host descriptors -> K4 -> K2 -> host results
    e2e = None
    n_ev_local = int(db.n_events)
    if not args.no_e2e:
        del db                              # HBM for a fresh expansion per step
        torch.cuda.synchronize()
        tt = time.perf_counter()
        reps = max(1, min(args.steps, 3))
        for _ in range(reps):
            db2 = xm.expand_templates(pool, d["tpl"], d["b"], d["seed"], mc5.SWAP_THRESHOLD,
                                      capacity=d["capacity"], stream=stream, check=False)
            r2 = xm.simulate_batch(db2, cfg, stream, out=out)
            h2, _ = xm.peaks(r2)
            del db2
        dt = (time.perf_counter() - tt) / reps
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=_cdev(dev))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t[0])
        T = len(mine)
        e2e = {"value": done / dt, "unit": UNIT, "h2d_bytes_per_step": int(40 * T + 8),
               "d2h_bytes_per_step": int(64 * T), "ms_per_step": dt * 1e3,
               "api": "xm_expand_templates (descriptors host->device, events generated in HBM) "
                      "+ xm_simulate_batch + xm_peaks (results device->host)",
               "results_equal_device_path": bool((h2 == h).all())}
    clocks = sampler.stop()

    peak, peak_src = peaks_json()
    alg = 12 * local_done + 24 * len(mine) + 64 * len(mine)
    achieved = alg / (kern_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None, "kernel": "k_replay",
            "alg_bytes_per_launch": alg, "kernel_ms": kern_ms, "peak_source": peak_src,
            "note": "K2 is a serial integer state machine per trace (issue/latency-bound)"}
    k4 = {"kernel": "k_expand", "ms": k4_ms, "bound": "hbm",
          "achieved": 12 * n_ev_local / (k4_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
          "frac": 12 * n_ev_local / (k4_ms / 1e3) / 1e9 / peak,
          "alg_bytes_per_launch": 12 * n_ev_local}
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.no_parity:
        # EVERY trace (north_star: bit-exact "for every trace versus the CPU
        # oracle"): forked workers rebuild their chunks on the host
        # (workloads/mc5gen.c, the documented recipe), replay them with the
        # oracle and compare all 13 fields with the GPU's results
        op = _oracle_pool()
        s = op.parity_mc5(np.arange(n), h)
        parity = {"traces": s["traces"], "fields": s["fields"],
                  "mismatched_values": s["mismatched_values"],
                  "mismatched_by_field": s["mismatched_by_field"],
                  "first_mismatch_trace": s["first_mismatch_trace"],
                  "sample": f"all {n} traces, host-built independently of K4",
                  "oracle_oom_traces": s["oracle_oom_traces"], "wall_s": s["wall_s"]}
        cpu = {"value": s["oracle_events"] / s["oracle_simulate_s_max_worker"], "unit": UNIT,
               "cores": s["workers"], "kind": "oracle", "cpu_model": op.cpu_model(),
               "sample": f"all {n} traces ({s['oracle_events']} replayed events); busiest of "
                         f"{s['workers']} forked workers simulated for "
                         f"{s['oracle_simulate_s_max_worker']:.1f} s (host trace generation "
                         f"excluded)",
               "wall_s_incl_generation_and_compare": s["wall_s"]}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        k = max(1, int(np.ceil(n_ev_local / 25_000_000)))
        sub = np.arange(0, n, k)
        hb = mc5.batch_fast(sub)
        rate, det, o = oracle_rate(hb)
        cpu = {"value": rate, "unit": UNIT, "cores": det["cores"], "kind": "oracle",
               "cpu_model": det["cpu_model"],
               "sample": f"every {k}th trace: {hb.n_traces} traces ({hb.n_events} events)"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic",
            "config": {"workload": f"configs[4] Monte Carlo: {n} perturbed traces generated on "
                                   f"device (K4), LPT-sharded over {world} GPU(s)",
                       "n_traces": n, "n_events": int(L.sum()), "events_done": done,
                       "traces_per_s": n / (ms / 1e3),
                       "l2": f"inputs larger than L2 ({12 * n_ev_local / 2**30:.1f} GiB/GPU)",
                       "parallelism": f"dp{world} (trace-sharded)",
                       "n_oom": summ["n_oom"], "n_overflow": summ["n_overflow"]},
            "gpu_launches": launches * args.steps, "roofline": roof, "k4_expand": k4,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "parity": parity}
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(s + "\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
