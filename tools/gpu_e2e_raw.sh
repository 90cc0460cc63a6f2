# xm_simulate_raw on config 4: GPU tests of the raw path, its time with the
# chunked DMA input (default) and reading in place (XM_RAW_INPUT=direct), the
# plain DMA copy, and the kernel launch list.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_raw.py -x -q 2>&1 | tail -2
timeout 300 python tools/e2e_raw_breakdown.py
XM_RAW_INPUT=direct timeout 300 python tools/e2e_raw_breakdown.py
REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/e2e_raw_breakdown.py 2>&1 | grep -E "k_" | awk -F'","' '{print $5, $NF}' | tail -4
