mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build3.log 2>&1 || tail -20 gpurun_out/build3.log
timeout 900 python -m pytest tests/test_gpu_k1_paths.py -x -q 2>&1 | tail -15
for p in c t f; do XM_K1=$p timeout 120 python tools/k1_stats.py cfg4 1; done
XM_K1=c timeout 120 python tools/k1_stats.py cfg4 8
XM_K1=t timeout 120 python tools/k1_stats.py cfg4 8
timeout 300 python tools/k2_stats.py cfg4 14
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_scan_chunks -s 2 -c 1 -o gpurun_out/prof/k_scan_chunks python tools/k1_stats.py cfg4 1 > /dev/null 2>&1; ls gpurun_out/prof
