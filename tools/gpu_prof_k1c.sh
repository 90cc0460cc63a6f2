mkdir -p gpurun_out/prof
XM_K1C_PER=8 XM_K1C_STAGES=2 XM_K1C_CTAS_PER_SM=4 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
XM_K1=c timeout 120 python tools/k1_stats.py cfg4 1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_scan_chunks -s 2 -c 1 -o gpurun_out/prof/k_scan_chunks2 python tools/k1_stats.py cfg4 1 > gpurun_out/prof/ncu_k1c.log 2>&1
XM_K1=t timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_scan_trace -s 2 -c 1 -o gpurun_out/prof/k_scan_trace python tools/k1_stats.py cfg4 1 > gpurun_out/prof/ncu_k1t.log 2>&1
ls gpurun_out/prof
