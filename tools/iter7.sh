python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_orchestrate.py -x -q 2>&1 | tail -2
timeout 900 python tools/bench_next.py orchestrate 2>&1 | grep '^{'
