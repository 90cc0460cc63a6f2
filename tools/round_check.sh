set -x
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 3 -c 1 -o gpurun_out/prof/k_replay python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_k2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_tiles -s 2 -c 1 -o gpurun_out/prof/k_scan_tiles python tools/k1_stats.py cfg4 8 > gpurun_out/prof/ncu_k1.log 2>&1
ls gpurun_out/prof
