#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "allocated_only" 2>&1 | tail -30
