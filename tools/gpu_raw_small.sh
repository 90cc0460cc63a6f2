python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_raw.py -x -q 2>&1 | grep -E "passed|failed" | tail -1
for w in cfg1 cfg2 cfg3; do
  for m in 1 0; do
    XM_RAW_OVERLAP=$m timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$w overlap=$m', 'e2e %.3f ms'%d['e2e']['ms_per_step'], 'dev %.3f ms'%d['ms_per_step'])"
  done
done
