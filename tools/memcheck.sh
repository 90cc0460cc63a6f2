python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -x -q -k "hand_traces" > gpurun_out/memcheck.log 2>&1
head -60 gpurun_out/memcheck.log
