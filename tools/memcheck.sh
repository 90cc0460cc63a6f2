timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python -m pytest tests/test_gpu_parity.py -x -q -k "spec1_fuzz" > gpurun_out/memcheck.log 2>&1
grep -v "Host Frame" gpurun_out/memcheck.log | head -40
