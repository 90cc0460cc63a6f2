# xm_simulate_raw: the landed-chunks count published after every n-th chunk
# (fewer stream memory operations between the copies) x number of chunks.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_raw.py -x -q 2>&1 | grep -E "passed|failed" | tail -1
med() { python -c "import json,sys,statistics as s; d=json.loads(sys.stdin.read()); print('median %.2f ms  min %.2f' % (s.median(d['simulate_raw_ms']), min(d['simulate_raw_ms'])))"; }
for r in 1 2; do
  for c in 48 96; do for f in 1 4 8; do
    echo "chunks=$c every=$f: $(XM_RAW_CHUNKS=$c XM_RAW_FLAG_EVERY=$f REPS=9 timeout 120 python tools/e2e_raw_breakdown.py | med)"
  done; done
done
XM_RAW_FLAG_EVERY=4 timeout 120 python tools/e2e_raw_timeline.py 2>&1 | tail -5
