#!/bin/bash
# deeper packed prefetch: parity (packed + host modes) and HBM vs host-read kernel times
set -e
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed or host_entry or config4" 2>&1 | tail -2
python tools/e2e_probe.py
PACKED=1 python tools/k2_stats.py cfg4 14
