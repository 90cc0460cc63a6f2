# xm_simulate_raw: upload chunks alternating over two copy streams vs one
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "1 stream: $(timeout 900 python -m pytest tests/test_gpu_raw.py -x -q 2>&1 | grep -E 'passed|failed' | tail -1)"
echo "2 streams: $(XM_RAW_COPY_STREAMS=2 timeout 900 python -m pytest tests/test_gpu_raw.py -x -q 2>&1 | grep -E 'passed|failed' | tail -1)"
med() { python -c "import json,sys,statistics as s; d=json.loads(sys.stdin.read()); print('median %.2f ms  min %.2f  copy %.2f' % (s.median(d['simulate_raw_ms']), min(d['simulate_raw_ms']), min(d['dma_copy_raw_ms'])))"; }
for r in 1 2; do
  for c in 48 96; do for n in 1 2; do
    echo "chunks=$c streams=$n: $(XM_RAW_CHUNKS=$c XM_RAW_COPY_STREAMS=$n REPS=9 timeout 120 python tools/e2e_raw_breakdown.py | med)"
  done; done
done
XM_RAW_COPY_STREAMS=2 timeout 120 python tools/e2e_raw_timeline.py 2>&1 | tail -5
