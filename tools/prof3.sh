timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 1 -c 1 -o gpurun_out/prof_k_replay_v3 python tools/k2_stats.py cfg4 8 > gpurun_out/ncu_v3.log 2>&1
tail -2 gpurun_out/ncu_v3.log
