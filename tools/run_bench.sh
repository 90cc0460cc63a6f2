python tools/k2_stats.py cfg4 8,10,12,14,16 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -c 2200 gpurun_out/bench.log
