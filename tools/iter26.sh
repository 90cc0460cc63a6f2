#!/bin/bash
# K1t claim-ahead: parity, then timing with and without (XM_K1_AHEAD)
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "allocated_only" 2>&1 | tail -2
for a in 1 0 1 0; do
  XM_K1_AHEAD=$a python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null
  echo "ahead $a"
  python tools/k1_stats.py cfg4 1
  python tools/k1_stats.py cfg4 8
done
