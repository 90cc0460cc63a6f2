mkdir -p gpurun_out/prof
XM_K1C_PER=16 XM_K1C_STAGES=2 XM_K1C_CTAS_PER_SM=2 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 300 python tools/k2_stats.py cfg4 14
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_scan_chunks -s 2 -c 1 -o gpurun_out/prof/k_scan_chunks python tools/k1_stats.py cfg4 1 > gpurun_out/prof/ncu_k1c.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 3 -c 1 -o gpurun_out/prof/k_replay_part python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_k2p.log 2>&1
ls gpurun_out/prof
