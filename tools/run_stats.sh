python tools/k2_stats.py cfg4 8,12,16 2>&1 | tail -3
