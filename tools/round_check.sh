# The round's GPU check: smoke, the GPU test suite, the bench lines, the ncu
# launch list and one full ncu capture per kernel (summarised into profiles/).
set -x
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 3500 gpurun_out/bench.log
timeout 900 python bench.py --workload cfg5 --steps 3 --warmup 3 > gpurun_out/bench_cfg5.log 2>&1; tail -c 1500 gpurun_out/bench_cfg5.log
timeout 900 python tools/bench_next.py > gpurun_out/bench_next.jsonl 2> gpurun_out/bench_next.err; cut -c1-300 gpurun_out/bench_next.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 3 -c 1 -o gpurun_out/prof/k_replay python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_k2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_trace -s 1 -c 1 -o gpurun_out/prof/k_scan_trace python tools/k1_stats.py cfg4 1 > gpurun_out/prof/ncu_k1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_reconstruct -s 1 -c 1 -o gpurun_out/prof/k_reconstruct python tools/bench_next.py lifecycle > gpurun_out/prof/ncu_k5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_orchestrate -s 1 -c 1 -o gpurun_out/prof/k_orchestrate python tools/bench_next.py orchestrate > gpurun_out/prof/ncu_k6.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_expand -s 1 -c 1 -o gpurun_out/prof/k_expand python tools/bench_next.py k4 > gpurun_out/prof/ncu_k4.log 2>&1
ls gpurun_out/prof
