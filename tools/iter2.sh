python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_lifecycle.py tests/test_gpu_config5.py -x -q 2>&1 | tail -3
timeout 900 python tools/bench_next.py lifecycle k4 2>&1 | grep '^{'
