#!/bin/bash
# K6: serial pass assigns ids only; sizes/streams gathered CTA-wide
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_orchestrate.py tests/test_gpu_pipeline.py -q -x 2>&1 | tail -2
timeout 900 python tools/bench_next.py orchestrate pipeline 2>&1 | grep '^{' | cut -c1-260
