python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/e2e_raw_timeline.py 2>&1 | tail -80
