python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config5.py -x -q 2>&1 | tail -2
python tools/k2_stats.py cfg4 10,12,14
python tools/k2_subset.py resnet152/adamw/pos1/b600/r0 1
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize.py > gpurun_out/sanitize_racecheck.log 2>&1; grep -E "RACECHECK SUMMARY|done" gpurun_out/sanitize_racecheck.log
