# K2 lean layout: parity first (the replay parity + K1 + raw suites), then A/B vs the previous layout.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/lean_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_raw.py tests/test_gpu_pipeline.py -x -q > gpurun_out/lean_parity.log 2>&1; tail -5 gpurun_out/lean_parity.log
timeout 900 bash tools/ab_k2.sh > gpurun_out/lean_ab.log 2>&1; cat gpurun_out/lean_ab.log
