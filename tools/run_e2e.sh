# streamed vs serial host entry point (xm_simulate_host), plus the GPU tests
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/e2e_streamed.json 2> gpurun_out/e2e_streamed.err
XM_NO_STREAM=1 python bench.py --no-cpu-baseline > gpurun_out/e2e_serial.json 2> gpurun_out/e2e_serial.err
python - <<'P'
import json
for f in ("streamed", "serial"):
    d = json.load(open(f"gpurun_out/e2e_{f}.json"))
    print(f, "kernel ms", d["ms_per_step"], "e2e ms", d["e2e"]["ms_per_step"], "e2e", d["e2e"]["value"])
P
