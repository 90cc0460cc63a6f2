# GPU parity tests + debug-build hand/fuzz run + K2 timing on config 4 + the bench line
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
XM_DEBUG=1 SPW=2048 timeout 300 python tools/debug_run.py 2>&1 | tail -2
XM_DEBUG=1 timeout 300 python tools/debug_run.py 2>&1 | tail -2
python tools/k2_stats.py cfg4 12,16
python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python - <<'P'
import json
d = json.load(open("gpurun_out/bench_quick.json"))
print("kernel ms", d["ms_per_step"], "value", d["value"], "e2e ms", d["e2e"]["ms_per_step"], "e2e", d["e2e"]["value"], "e2e==dev", d["e2e"].get("results_equal_device_path"))
P
