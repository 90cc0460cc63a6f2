# one optimisation iteration on the box: build, GPU parity tests, K2 geometry sweep, bench (no CPU baseline)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/k2_stats.py cfg4 ${WPC:-12,16}
python tools/k2_subset.py resnet152/adamw/pos1/b600/r0 1
timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python - <<'P'
import json
d = json.load(open("gpurun_out/bench_quick.json"))
print("kernel ms", d["ms_per_step"], "value %.3e" % d["value"], "e2e ms", d["e2e"]["ms_per_step"], "e2e %.3e" % d["e2e"]["value"], "parity", d.get("parity"), "clocks", d.get("clocks"))
P
