python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "heap_page" 2>&1 | grep -v Warning | tail -5
