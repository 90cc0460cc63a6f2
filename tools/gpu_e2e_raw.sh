# xm_simulate_raw on config 4: GPU tests of the raw path, its time with the
# chunked DMA input (default) and reading in place (XM_RAW_INPUT=direct), and
# a CUPTI timeline of one call.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_raw.py -x -q 2>&1 | tail -2
timeout 300 python tools/e2e_raw_breakdown.py
XM_RAW_INPUT=direct timeout 300 python tools/e2e_raw_breakdown.py
timeout 300 python tools/e2e_raw_timeline.py 2>&1 | grep -E "k_|Memcpy DtoH" | tail -8
