# smoke, the GPU suite, and the driver-style bench lines for configs 1-3
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; tail -1 gpurun_out/final/pytest_gpu.log
for w in cfg1 cfg2 cfg3; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/final/bench_$w.log 2>&1; tail -1 gpurun_out/final/bench_$w.log > gpurun_out/final/r02_bench_$w.json; done
ls gpurun_out/final
