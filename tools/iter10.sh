python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json')); print('kernel', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], d['e2e']['h2d_bytes_per_step'], d['e2e']['results_equal_device_path'], 'K1', d['roofline_k1_allocated_only']['ms'])"; done
