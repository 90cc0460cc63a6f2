python tools/k2_stats.py cfg4 1,2,4,8,16 2>&1 | tail -8
