python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
python tools/k2_stats.py cfg4 12
python tools/k2_stats.py cfg4 12
python tools/k2_subset.py resnet152/adamw/pos1/b600/r0 1
