#!/bin/bash
# K5 tables sized by n/2 with regrow-and-restart: parity, then timing
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_lifecycle.py tests/test_gpu_pipeline.py -q -x 2>&1 | tail -2
timeout 900 python tools/bench_next.py lifecycle pipeline 2>&1 | grep '^{' | cut -c1-300
