set -x
XM_DEBUG=1 timeout 120 python tools/debug_run.py all > gpurun_out/debug_all.log 2>&1; tail -3 gpurun_out/debug_all.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; cat gpurun_out/smoke.log | tail -2
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -c 2500 gpurun_out/bench.log
