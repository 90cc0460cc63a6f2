mkdir -p gpurun_out/prof
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof/k1_launches.csv python tools/k1_stats.py cfg4 8 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_tiles -s 2 -c 1 -o gpurun_out/prof/k_scan_tiles_v4 python tools/k1_stats.py cfg4 8 > gpurun_out/prof/ncu_k1.log 2>&1
tail -1 gpurun_out/prof/ncu_k1.log
