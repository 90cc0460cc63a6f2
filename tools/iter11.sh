python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "allocated_only or packed" 2>&1 | tail -1
python tools/k1_stats.py cfg4 1 2>&1 | tail -1
python tools/k1_stats.py cfg4 1 2>&1 | tail -1
