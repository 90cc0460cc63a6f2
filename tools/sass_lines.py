"""Aggregate an ncu SASS source page (CSV) by CUDA source line, using the
line table nvdisasm -g prints for the same (locally rebuilt, identical) cubin.

usage: python tools/sass_lines.py NCU_SASS.csv NVDISASM.sass FUNC_SUBSTR [TOP]
"""
import csv, re, sys, collections
csv_path, sass_path, func = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
# offset -> (file line) from nvdisasm
lines = {}          # offset -> innermost (file, line); chains -> every line of the inline chain
chains = {}
chain = []
inside = False
pending = False
for ln in open(sass_path):
    if ln.startswith("//---------------------"):
        inside = func in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
    if m:
        if not pending:
            chain = []
        pending = True
        if not chain:
            chain.append((m.group(1).split("/")[-1], int(m.group(2))))
        if m.group(3):
            chain.append((m.group(3).split("/")[-1], int(m.group(4))))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        pending = False
        off = int(m.group(1), 16)
        lines[off] = chain[0] if chain else None
        chains[off] = list(chain)
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ia = hdr.index("Address"); ie = hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)"); isrc = hdr.index("Source")
data = rows[2:]
base = int(data[0][ia], 16)
agg = collections.defaultdict(lambda: [0, 0, ""])
tot_i = tot_s = 0
for r in data:
    off = int(r[ia], 16) - base
    key = lines.get(off)
    k = f"{key[0]}:{key[1]}" if key else "?"
    if key and len(key) > 2:
        k += f" (in {key[2][0]}:{key[2][1]})"
    n = int(r[ie].replace(",", "") or 0); s = int(r[iss].replace(",", "") or 0)
    agg[k][0] += n; agg[k][1] += s
    tot_i += n; tot_s += s
print(f"total warp-inst {tot_i:.4g}  stall samples {tot_s}")
for k, (n, s, _) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{100*n/tot_i:6.2f}% inst  {100*s/tot_s:6.2f}% stall  {k}")

# stall-reason totals and per-region breakdown
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for r in data:
    for h in reasons:
        v = r[hdr.index(h)].replace(",", "")
        tot[h] += int(v or 0)
S = sum(tot.values())
print("stall reasons:", ", ".join(f"{h[6:]} {100*v/S:.1f}%" for h, v in tot.most_common(10)))
if len(sys.argv) > 5:
    regions = eval(sys.argv[5])   # {"name": (lo, hi), ...} source-line ranges of the main file
    reg = collections.defaultdict(lambda: [0, 0])
    for r in data:
        off = int(r[ia], 16) - base
        name = "other"
        for (f, ln) in chains.get(off, []):
            hit = next((nm for nm, (lo, hi) in regions.items() if f == "replay.cu" and lo <= ln <= hi), None)
            if hit:
                name = hit
                break
        reg[name][0] += int(r[ie].replace(",", "") or 0)
        reg[name][1] += int(r[iss].replace(",", "") or 0)
    for nm, (n, s) in sorted(reg.items(), key=lambda kv: -kv[1][0]):
        print(f"{nm:14s} {100*n/tot_i:6.2f}% inst {100*s/tot_s:6.2f}% stall")
