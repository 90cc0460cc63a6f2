mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 0 296 148 74 37; do
  if [ $c = 0 ]; then unset XM_K5_CTAS; else export XM_K5_CTAS=$c; fi
  timeout 300 python tools/k5_sweep.py
  REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_reconstruct -c 1 --csv python tools/k5_sweep.py 2>/dev/null | grep -E "k_reconstruct" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
