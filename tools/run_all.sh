XM_DEBUG=1 timeout 120 python tools/debug_run.py all > gpurun_out/debug_all.log 2>&1; tail -1 gpurun_out/debug_all.log | cut -c1-300
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python tools/k2_stats.py cfg4 1,8,12,16 2>&1 | tail -4
