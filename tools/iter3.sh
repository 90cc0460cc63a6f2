python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "allocated_only" 2>&1 | tail -2
python tools/k1_stats.py cfg4 1 2>&1 | tail -1
python tools/k1_stats.py cfg4 8 2>&1 | tail -1
python tools/k2_stats.py cfg4 12
timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json')); print(d['ms_per_step'], d['roofline_k1_allocated_only'])"
