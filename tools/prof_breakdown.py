"""Per-region instruction / stall breakdown of k_replay from an ncu report
(source page, --print-source cuda): python tools/prof_breakdown.py REPORT EVENTS"""
import csv, io, os, subprocess, sys
from collections import Counter
rep, EV = sys.argv[1], float(sys.argv[2])
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
ie = hdr.index("Instructions Executed")
smp = hdr.index("Warp Stall Sampling (All Samples)")
lines = {}
for r in rows[hi + 1:]:
    try:
        lines[int(r[0])] = (r[1][:90], float(r[ie] or 0), float(r[smp] or 0))
    except (ValueError, IndexError):
        pass
src = open(os.path.join(ROOT, "paper_2510_21048_b200/csrc/replay.cu")).read().split("\n")
def find(pat):
    return next(i + 1 for i, l in enumerate(src) if pat in l)
marks = [("tile+decode", "const int64_t bc = b_nx;"), ("scan+reduce", "================= ALLOC"),
         ("alloc load", "// ---- load phase (plus the rare reclaim"), ("alloc store", "        // ---- store phase ----"),
         ("free load", "================= FREE"), ("free store", "// ---- store phase: a8"),
         ("event end", "if (curve && lane == j)"), ("tile end", "    if (curve && lane < j)"),
         ("(after)", "  const uint32_t sh = u.unit_shift;")]
pos = [(n, find(p)) for n, p in marks]
tot = sum(v[1] for v in lines.values()); ts = sum(v[2] for v in lines.values())
print(f"total {tot / EV:.1f} warp-inst per event")
for k in range(len(pos) - 1):
    n, a = pos[k]; b = pos[k + 1][1]
    ins = sum(v[1] for l, v in lines.items() if a <= l < b); sm = sum(v[2] for l, v in lines.items() if a <= l < b)
    print(f"  {n:14s} {ins / EV:6.1f} inst/ev {sm / ts * 100:5.1f}% samples")
a, b = pos[0][1], pos[-1][1]
oth = [(l, v) for l, v in lines.items() if not (a <= l < b)]
print(f"  {'helpers/other':14s} {sum(v[1] for _, v in oth) / EV:6.1f} inst/ev {sum(v[2] for _, v in oth) / ts * 100:5.1f}% samples")
for l, v in sorted(oth, key=lambda x: -x[1][1])[:15]:
    print(f"     {l:5d} {v[1] / EV:6.2f}/ev {v[2] / ts * 100:5.1f}%  {v[0]}")
