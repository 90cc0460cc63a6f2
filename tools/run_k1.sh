timeout 600 python -m pytest tests -m gpu -q -x -k "allocated_only" 2>&1 | tail -1
python tools/k1_stats.py cfg4 1 2>&1 | tail -1
python tools/k1_stats.py cfg4 8 2>&1 | tail -1
python tools/k1_stats.py cfg4 24 2>&1 | tail -1
