#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
PACKED=1 python tools/k2_stats.py cfg4 14,14,15
python tools/e2e_probe.py
