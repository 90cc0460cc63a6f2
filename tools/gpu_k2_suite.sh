# the K2 parity suites (after a K2 change)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config5.py tests/test_gpu_raw.py tests/test_gpu_pipeline.py tests/test_torch_allocator_pin.py -x -q 2>&1 | tail -2
