# The round's GPU check: smoke, the GPU test suite, the bench lines (config 4
# default, config 5 with every-trace parity, configs 1-3), the widened rows,
# the ncu launch list and one full ncu capture per kernel, summarised into
# profiles/ (ncu_summary.json is read by bench.py for roofline.traffic/issue:
# the bench runs once more after the summary is written).
set -x
mkdir -p gpurun_out/prof gpurun_out/round
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/round/smoke.log 2>&1; tail -1 gpurun_out/round/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/round/pytest_gpu.log 2>&1; tail -2 gpurun_out/round/pytest_gpu.log
timeout 300 python tools/e2e_raw_timeline.py > gpurun_out/round/raw_timeline.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-k1 > gpurun_out/prof/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 3 -c 1 -o gpurun_out/prof/k_replay python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_k2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_trace -s 2 -c 1 -o gpurun_out/prof/k_scan_trace env XM_K1=t python tools/k1_stats.py cfg4 1 > gpurun_out/prof/ncu_k1t.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_chunks -s 2 -c 1 -o gpurun_out/prof/k_scan_chunks env XM_K1=c python tools/k1_stats.py cfg4 1 > gpurun_out/prof/ncu_k1c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_reconstruct -s 1 -c 1 -o gpurun_out/prof/k_reconstruct python tools/bench_next.py lifecycle > gpurun_out/prof/ncu_k5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_orchestrate -s 1 -c 1 -o gpurun_out/prof/k_orchestrate python tools/bench_next.py orchestrate > gpurun_out/prof/ncu_k6.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_expand -s 1 -c 1 -o gpurun_out/prof/k_expand python tools/bench_next.py k4 > gpurun_out/prof/ncu_k4.log 2>&1
# k_load on the sequential raw path (ncu serialises kernels; the overlapped
# loader and replay wait on each other, so they cannot be profiled together)
XM_RAW_OVERLAP=0 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_load -s 1 -c 1 -o gpurun_out/prof/k_load python tools/e2e_raw_breakdown.py > gpurun_out/prof/ncu_kload.log 2>&1
python tools/ncu_summary.py 02 k_replay=gpurun_out/prof/k_replay.ncu-rep k_scan_trace=gpurun_out/prof/k_scan_trace.ncu-rep \
  k_scan_chunks=gpurun_out/prof/k_scan_chunks.ncu-rep k_reconstruct=gpurun_out/prof/k_reconstruct.ncu-rep \
  k_orchestrate=gpurun_out/prof/k_orchestrate.ncu-rep k_expand=gpurun_out/prof/k_expand.ncu-rep \
  k_load=gpurun_out/prof/k_load.ncu-rep \
  --launches gpurun_out/prof/launches.csv > gpurun_out/round/ncu_summary.log 2>&1
cp profiles/ncu_summary.json profiles/r02_ncu_summary.md gpurun_out/round/ 2>/dev/null
cp gpurun_out/prof/launches.csv gpurun_out/round/r02_launches.csv
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/round/bench.log 2>&1; tail -1 gpurun_out/round/bench.log > gpurun_out/round/r02_bench.json
timeout 1200 python bench.py --workload cfg5 --steps 3 --warmup 3 > gpurun_out/round/bench_cfg5.log 2>&1; tail -1 gpurun_out/round/bench_cfg5.log > gpurun_out/round/r02_bench_cfg5.json
for w in cfg1 cfg2 cfg3; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/round/bench_$w.log 2>&1; tail -1 gpurun_out/round/bench_$w.log > gpurun_out/round/r02_bench_$w.json; done
timeout 900 python tools/bench_next.py > gpurun_out/round/r02_bench_next.jsonl 2> gpurun_out/round/bench_next.err
ls -la gpurun_out/round
