# smoke + the whole GPU suite + the default bench line
mkdir -p gpurun_out/full
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/full/smoke.log 2>&1; tail -1 gpurun_out/full/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/full/pytest_gpu.log 2>&1; tail -2 gpurun_out/full/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/full/bench.log 2>&1; tail -1 gpurun_out/full/bench.log > gpurun_out/full/bench.json
python -c "import json; d=json.load(open('gpurun_out/full/bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['parity'], d['roofline_k1_allocated_only']['frac'])"
