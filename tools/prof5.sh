mkdir -p gpurun_out/prof
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 1 -c 1 -o gpurun_out/prof/k_replay_w12 -f python tools/k2_stats.py cfg4 12 > /dev/null 2>&1
ls gpurun_out/prof
