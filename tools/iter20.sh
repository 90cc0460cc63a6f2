python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_lifecycle.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -1
timeout 900 python tools/bench_next.py lifecycle pipeline 2>&1 | grep '^{' | cut -c1-330
