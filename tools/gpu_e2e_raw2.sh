python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_raw.py tests/test_gpu_parity.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -2
timeout 300 python tools/e2e_raw_breakdown.py
timeout 300 python tools/e2e_raw_timeline.py 2>&1 | grep -E "k_|Memcpy DtoH" | tail -8
