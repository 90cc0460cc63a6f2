python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/e2e_raw_breakdown.py
REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/e2e_raw_breakdown.py 2>&1 | grep -E "k_|Kernel|duration" | tail -30
