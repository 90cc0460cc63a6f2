"""Measurement of the NEXT rows (one JSON line each, GPU box):

  lifecycle  K5 xm_reconstruct on config-4-shaped profiler instants (5209
             traces, ~29M instants, addresses with reuse + noise), device-
             resident: instants/s, roofline (34 algorithmic B/instant: 17 read,
             17 written), and the chained instants -> reconstruct -> replay
             (K5 + K2) time; the oracle on host cores on a sample.
  metrics    xm_metrics_batch on 1M run records.
  k4         K4 expansion of config 5 (1M traces): GB/s of the 12 B/event writes.

usage: python tools/bench_next.py [lifecycle|metrics|k4 ...]
"""
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _inst_part(args):
    from workloads import instants, suites
    lo, hi = int(args[0]), int(args[1])
    b = suites.config4()
    return instants.from_batch(b.subset(range(lo, hi)), salt=4 + lo, p_orphan=0.001,
                               p_mismatch=0.001, p_lost=0.002)


def _time(fn, reps, torch):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def lifecycle():
    import torch
    import paper_2510_21048_b200 as xm
    from workloads import instants
    t0 = time.time()
    cuts = np.linspace(0, 5209, 33).astype(int)
    with Pool(min(32, os.cpu_count() or 4)) as pool:
        parts = pool.map(_inst_part, list(zip(cuts[:-1], cuts[1:])))
    off = [np.zeros(1, np.int64)]
    base = 0
    for p in parts:
        off.append(p.off[1:] + base)
        base += p.n_events
    ins = instants.Instants(np.concatenate([p.addr for p in parts]),
                            np.concatenate([p.bytes for p in parts]),
                            np.concatenate([p.stream for p in parts]), np.concatenate(off))
    gen_s = time.time() - t0
    d = xm.DeviceInstants.from_host(ins.addr, ins.bytes, ins.stream, ins.off)
    scratch = torch.empty(int(xm.lib().xm_reconstruct_scratch_bytes(__import__("ctypes").byref(d.c()))),
                          dtype=torch.uint8, device="cuda")
    ms_nowire = _time(lambda: xm.reconstruct(d, wire=False, scratch=scratch), 5, torch)
    ms_wire = _time(lambda: xm.reconstruct(d, wire=True, scratch=scratch), 5, torch)
    _, _, rec, wb = xm.reconstruct(d, scratch=scratch)
    out = torch.empty((wb.n_traces, 64), dtype=torch.uint8, device="cuda")
    ms_replay = _time(lambda: xm.simulate_batch(wb, out=out), 5, torch)
    ms_chain = _time(lambda: xm.simulate_batch(xm.reconstruct(d, scratch=scratch)[3], out=out), 3, torch)
    E = ins.n_events
    peak, psrc = _peak()
    alg = 34 * E
    ach = alg / (ms_wire / 1e3) / 1e9
    # oracle on a sample (host cores)
    import oracle
    k = 10
    t1 = time.time()
    n_s = 0
    for t in range(0, ins.n_traces, k):
        a, by, st = ins.trace(t)
        oracle.reconstruct(a, by)
        n_s += len(by)
    cpu_rate = n_s / (time.time() - t1)
    return {"row": "NEXT-3 lifecycle reconstruction (xm_reconstruct, K5)",
            "workload": f"config-4-shaped instants: {ins.n_traces} traces, {E} instants "
                        f"(host generation {gen_s:.1f} s)",
            "instants_per_s": E / (ms_wire / 1e3), "ms": ms_wire, "ms_without_wire": ms_nowire,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "alg_bytes_per_launch": alg, "peak_source": psrc},
            "chain_instants_to_peaks_ms": ms_chain, "replay_ms": ms_replay,
            "tallies": {k: int(rec[k].sum()) for k in ("n_blocks", "n_orphan", "n_mismatch",
                                                      "n_persistent", "n_kept")},
            "cpu_baseline": {"value": cpu_rate, "unit": "instants/s", "cores": 1, "kind": "oracle",
                             "sample": f"every {k}th trace, {n_s} instants, single thread"}}


def _prof_part(args):
    from workloads import cpu_profile as C
    lo, hi = int(args[0]), int(args[1])
    cells = C.suite_cells(hi)[lo:hi]
    return C.batch(cells, salt=20 + lo)


def orchestrate():
    import torch
    import paper_2510_21048_b200 as xm
    from workloads import cpu_profile as C
    n = 5209
    t0 = time.time()
    cuts = np.linspace(0, n, 33).astype(int)
    with Pool(min(32, os.cpu_count() or 4)) as pool:
        parts = pool.map(_prof_part, list(zip(cuts[:-1], cuts[1:])))
    boff, woff = [np.zeros(1, np.int64)], [np.zeros(1, np.int64)]
    bb = wb_ = 0
    for p in parts:
        boff.append(p.boff[1:] + bb)
        woff.append(p.woff[1:] + wb_)
        bb += int(p.boff[-1])
        wb_ += int(p.woff[-1])
    cat = lambda k: np.concatenate([getattr(p, k) for p in parts])
    prof = C.Profiles(cat("alloc_ts"), cat("free_ts"), cat("size"), cat("stream"), cat("kind"),
                      np.concatenate(boff), cat("win"), np.concatenate(woff))
    gen_s = time.time() - t0
    d = xm.DeviceProfiles.from_host(prof)
    import ctypes
    scratch = torch.empty(int(xm.lib().xm_orchestrate_scratch_bytes(ctypes.byref(d.c()))),
                          dtype=torch.uint8, device="cuda")
    ms = _time(lambda: xm.orchestrate(d, wire=False, scratch=scratch), 5, torch)
    ms_wire = _time(lambda: xm.orchestrate(d, wire=True, scratch=scratch), 3, torch)
    _, _, rec, wb = xm.orchestrate(d, scratch=scratch)
    out = torch.empty((wb.n_traces, 64), dtype=torch.uint8, device="cuda")
    ms_replay = _time(lambda: xm.simulate_batch(wb, out=out), 5, torch)
    B = int(prof.boff[-1])
    peak, psrc = _peak()
    # algorithmic bytes: read 33 B/block (alloc, free, size, stream) + windows,
    # write 1 B class + 8 B per sequence key
    n_ev = int(rec["n_events"].sum())
    alg = 33 * B + 8 * int(prof.win.size) + B + 8 * n_ev + 56 * prof.n_traces
    ach = alg / (ms / 1e3) / 1e9
    from oracle import orchestrator as O
    k = 20
    t1 = time.time()
    nb = 0
    for t in range(0, prof.n_traces, k):
        a, f, s, st, W = prof.trace(t)
        O.orchestrate(a, f, s, W)
        nb += len(a)
    cpu = nb / (time.time() - t1)
    return {"row": "NEXT-2 memory orchestrator (xm_orchestrate, K6)",
            "workload": f"{prof.n_traces} Monte-Carlo-drawn CPU profiles, {B} blocks, "
                        f"{n_ev} re-timed events (host generation {gen_s:.1f} s)",
            "blocks_per_s": B / (ms / 1e3), "ms": ms, "ms_with_wire": ms_wire,
            "replay_of_orchestrated_ms": ms_replay,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "alg_bytes_per_launch": alg, "peak_source": psrc,
                         "note": "per-trace CTA with an O(C(C+P)) quota count and a bitonic "
                                 "sort: compute/latency-bound, not HBM-bound"},
            "cpu_baseline": {"value": cpu, "unit": "blocks/s", "cores": 1, "kind": "oracle",
                             "sample": f"every {k}th trace, {nb} blocks, single thread (Python)"}}


def _pipe_part(args):
    from workloads import cpu_profile as C
    lo, hi = int(args[0]), int(args[1])
    p = C.batch(C.suite_cells(hi)[lo:hi], salt=40 + lo)
    return p, C.to_instants(p)


def pipeline():
    """Profiler instants (with times and annotation windows) -> estimated
    peaks, all on the GPU (xm.estimate: K5 -> blocks -> K6 -> K2)."""
    import torch
    import paper_2510_21048_b200 as xm
    n = 5209
    t0 = time.time()
    cuts = np.linspace(0, n, 33).astype(int)
    with Pool(min(32, os.cpu_count() or 4)) as pool:
        parts = pool.map(_pipe_part, list(zip(cuts[:-1], cuts[1:])))
    ts = np.concatenate([q[1][0] for q in parts])
    ad = np.concatenate([q[1][1] for q in parts])
    by = np.concatenate([q[1][2] for q in parts])
    st = np.concatenate([q[1][3] for q in parts])
    off, woff, base, wb_ = [np.zeros(1, np.int64)], [np.zeros(1, np.int64)], 0, 0
    for prof, ins in parts:
        off.append(ins[4][1:] + base)
        base += int(ins[4][-1])
        woff.append(prof.woff[1:] + wb_)
        wb_ += int(prof.woff[-1])
    off = np.concatenate(off)
    woff = np.concatenate(woff)
    win = np.concatenate([q[0].win for q in parts])
    gen_s = time.time() - t0
    d = xm.DeviceInstants.from_host(ad, by, st, off)
    d_ts = torch.from_numpy(ts).cuda()
    caps = np.full(n, 12 << 30, np.uint64)
    ms = _time(lambda: xm.estimate(d, d_ts, win, woff, capacity=caps), 3, torch)
    h, summ, det = xm.estimate(d, d_ts, win, woff, capacity=caps)
    return {"row": "GPU pipeline: instants -> reconstruct -> orchestrate -> replay (xm.estimate)",
            "workload": f"{n} Monte-Carlo-drawn CPU profiles as {len(by)} profiler instants "
                        f"(host generation {gen_s:.1f} s), 12 GiB capacity",
            "ms": ms, "instants_per_s": len(by) / (ms / 1e3), "traces_per_s": n / (ms / 1e3),
            "n_oom": summ["n_oom"],
            "note": "includes the host syncs between the stages (per-trace records are read to "
                    "size the next stage)"}


def metrics():
    import torch
    import paper_2510_21048_b200 as xm
    rng = np.random.default_rng(0)
    n = 1_000_000
    GiB = 1 << 30
    r = np.zeros(n, xm.RUN_DTYPE)
    r["m_max"] = rng.choice([8 * GiB, 12 * GiB], n)
    r["m_peak_est"] = rng.integers(1, 2 * r["m_max"].astype(np.int64))
    r["oom_pred"] = r["m_peak_est"] > r["m_max"]
    r["oom1"] = rng.random(n) < 0.3
    run2 = (r["oom_pred"] == r["oom1"]) & (r["oom1"] == 0)
    r["oom2"] = np.where(run2, rng.random(n) < 0.2, 2)
    r["m_peak_meas1"] = rng.integers(1, r["m_max"].astype(np.int64))
    r["m_peak_meas2"] = rng.integers(1, r["m_max"].astype(np.int64))
    d = torch.from_numpy(r.view(np.uint8).reshape(-1, 40)).cuda()
    xm.metrics(d)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        m = xm.metrics(d)
    dt = (time.perf_counter() - t0) / 5
    return {"row": "NEXT-4 batched metrics (xm_metrics_batch)", "runs": n, "ms": dt * 1e3,
            "runs_per_s": n / dt, "mre": m["mre"], "pef2": m["pef2"], "mcp": m["mcp"]}


def k4():
    import torch
    import paper_2510_21048_b200 as xm
    from workloads import mc5
    n = 1_000_000
    d = mc5.describe(np.arange(n))
    pool = xm.Templates(*mc5.template_pool())
    db = xm.expand_templates(pool, d["tpl"], d["b"], d["seed"], mc5.SWAP_THRESHOLD)
    ms = _time(lambda: xm.expand_again(pool, db), 3, torch)
    peak, psrc = _peak()
    alg = 12 * db.n_events
    ach = alg / (ms / 1e3) / 1e9
    return {"row": "K4 config-5 expansion (xm_expand_templates)", "traces": n,
            "events": db.n_events, "ms": ms,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "alg_bytes_per_launch": alg, "peak_source": psrc}}


if __name__ == "__main__":
    which = sys.argv[1:] or ["lifecycle", "orchestrate", "pipeline", "metrics", "k4"]
    for w in which:
        try:
            print(json.dumps(globals()[w]()), flush=True)
        except Exception as e:  # report and go on with the next row
            import traceback
            traceback.print_exc()
            print(json.dumps({"row": w, "error": repr(e)}), flush=True)
