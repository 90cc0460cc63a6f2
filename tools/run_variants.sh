python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_torch_allocator_pin.py -x -q 2>&1 | tail -15
