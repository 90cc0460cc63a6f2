timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 1 -c 1 -o gpurun_out/prof_k_replay_w1 python tools/k2_stats.py cfg4 1 > gpurun_out/ncu_w1.log 2>&1
tail -2 gpurun_out/ncu_w1.log
