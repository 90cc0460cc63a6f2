for k in 16384 8192; do
  XM_ORCH_SMEM_KEYS=$k python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" || exit 1
  echo "== smem keys $k"; timeout 600 python -m pytest tests/test_gpu_orchestrate.py -x -q 2>&1 | tail -1
  timeout 900 python tools/bench_next.py orchestrate 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms'], d['ms_with_wire'])"
done
python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)"
