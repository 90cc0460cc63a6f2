# config 5 on the box: K4 parity tests + bench lines (1M traces and a small run)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_config5.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --workload cfg5 --steps 3 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
tail -c 3000 gpurun_out/bench_cfg5.json; tail -5 gpurun_out/bench_cfg5.err
