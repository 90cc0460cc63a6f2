"""Summarise ncu captures into profiles/ (tracked): ncu_summary.json (read by
bench.py for roofline.traffic) and a markdown table.

usage: python tools/ncu_summary.py ROUND KERNEL=REPORT.ncu-rep [KERNEL=REPORT ...]
       [--launches LAUNCHES.csv] [--units KERNEL=EVENTS_PER_LAUNCH ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_inst",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k, name in METRICS.items():
        col = next((i for i, h in enumerate(hdr) if h == k or h.endswith("." + k)), None)
        if col is not None:
            v = vals[col].replace(",", "")
            try:
                d[name] = float(v)
            except ValueError:
                d[name] = v
            u = units[col]
            if name == "duration_ns" and u in ("usecond", "us"):
                d[name] *= 1e3
            if name == "duration_ns" and u in ("msecond", "ms"):
                d[name] *= 1e6
            if name.startswith("dram_") and name.endswith("bytes"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                d[name] *= scale
    d["dram_bytes_per_launch"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
    if d.get("duration_ns"):
        d["dram_GBps"] = d["dram_bytes_per_launch"] / d["duration_ns"]
    return d


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    kn, mn, mv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[start + 1:]:
        if r[mn] != "gpu__time_duration.sum":
            continue
        name = r[kn].split("(")[0].replace("<unnamed>::", "")
        agg.setdefault(name, []).append(float(r[mv].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "mean_ns": sum(v) / len(v), "share": sum(v) / tot}
            for k, v in agg.items()}


def main():
    args = sys.argv[1:]
    rnd = args.pop(0)
    lpath = None
    units = {}
    reps = {}
    while args:
        a = args.pop(0)
        if a == "--launches":
            lpath = args.pop(0)
        elif a == "--units":
            k, v = args.pop(0).split("=")
            units[k] = float(v)
        else:
            k, v = a.split("=")
            reps[k] = v
    summ = {"round": rnd, "kernels": {}, "source": "ncu --set full --clock-control none"}
    for k, rep in reps.items():
        d = raw(rep)
        d["source"] = os.path.basename(rep)
        if k in units:
            d["units_per_launch"] = units[k]
            d["dram_bytes_per_unit"] = d["dram_bytes_per_launch"] / units[k]
        summ["kernels"][k] = d
    if lpath:
        summ["launch_list"] = launches(lpath)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
        json.dump(summ, f, indent=1, sort_keys=True)
    lines = [f"# ncu summary, round {rnd}", "",
             "| kernel | duration | DRAM bytes/launch | DRAM GB/s | % of measured HBM peak | issue active % | occupancy % | regs | warp inst |",
             "|---|---|---|---|---|---|---|---|---|"]
    def num(d, k):
        v = d.get(k, 0)
        return v if isinstance(v, float) else 0.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except Exception:
        hbm = 6650.0                       # B200_PROFILING.md fallback
    for k, d in summ["kernels"].items():
        d = {kk: (vv if not isinstance(vv, str) or kk == "source" else 0.0) for kk, vv in d.items()}
        d["dram_throughput_pct"] = 100.0 * d.get("dram_GBps", 0) / hbm
        lines.append(f"| {k} | {d.get('duration_ns', 0) / 1e6:.3f} ms | {d['dram_bytes_per_launch']:.4g} | "
                     f"{d.get('dram_GBps', 0):.0f} | "
                     f"{d.get('dram_throughput_pct', 0):.1f} | {d.get('issue_active_pct', 0):.1f} | "
                     f"{d.get('achieved_occupancy_pct', 0):.1f} | {d.get('registers_per_thread', 0):.0f} | "
                     f"{d.get('warp_instructions', 0):.4g} |")
    if lpath:
        lines += ["", "Launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised):", "",
                  "| kernel | launches | mean | share |", "|---|---|---|---|"]
        for k, d in summ["launch_list"].items():
            lines.append(f"| {k} | {d['launches']} | {d['mean_ns'] / 1e6:.3f} ms | {d['share'] * 100:.1f}% |")
    with open(os.path.join(ROOT, "profiles", f"r{rnd}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
