# xm_simulate_raw with the loader overlapped with the replay: the raw-path GPU
# tests, then config-4 e2e time vs the loader's SM count, the number of upload
# chunks, and the sequential path.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_raw.py -x -q 2>&1 | grep -E "passed|failed|Error" | tail -3
med() { python -c "import json,sys,statistics as s; d=json.loads(sys.stdin.read()); print('median %.2f ms  min %.2f' % (s.median(d['simulate_raw_ms']), min(d['simulate_raw_ms'])))"; }
echo "seq: $(XM_RAW_OVERLAP=0 REPS=7 timeout 120 python tools/e2e_raw_breakdown.py | med)"
for c in ${CHUNKS:-24 48 96 192}; do for s in ${SMS:-16 24 32}; do
  echo "chunks=$c sms=$s: $(XM_RAW_CHUNKS=$c XM_RAW_LOADER_SMS=$s REPS=7 timeout 120 python tools/e2e_raw_breakdown.py | med)"
done; done
