#!/bin/bash
# K1t geometry with the redux argmax (XM_K1_WARPS, XM_K1_PER_LANE)
for g in "4 8" "8 8" "4 16" "2 16" "8 4"; do
  set -- $g
  XM_K1_WARPS=$1 XM_K1_PER_LANE=$2 python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "warps $1 per_lane $2"
  python tools/k1_stats.py cfg4 1 | cut -c1-120
  python tools/k1_stats.py cfg4 8 | cut -c1-120
done
