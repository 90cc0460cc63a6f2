timeout 1200 python -m pytest tests/test_torch_allocator_pin.py -q -x 2>&1 | tail -25
