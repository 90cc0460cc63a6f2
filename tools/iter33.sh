#!/bin/bash
# metrics: grid-wide radix select
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_metrics.py -q -x 2>&1 | tail -2
timeout 900 python tools/bench_next.py metrics 2>&1 | grep '^{' | cut -c1-300
