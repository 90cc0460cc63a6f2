#!/bin/bash
# K1t warp argmax by 32-bit reductions: parity, then timing
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "allocated_only or variant" 2>&1 | tail -2
for i in 1 2; do python tools/k1_stats.py cfg4 1; python tools/k1_stats.py cfg4 8; done
