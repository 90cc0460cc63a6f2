python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
XM_TIMING=1 python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
timeout 120 python tools/e2e_raw_timeline.py 2>&1 | tail -8
timeout 120 python tools/k2_raw_timing.py 2>&1 | tail -20
