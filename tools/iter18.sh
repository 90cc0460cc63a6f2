for cfg in "4 8" "4 4" "8 4" "8 8" "2 8" "4 16"; do
  set -- $cfg
  XM_K1_WARPS=$1 XM_K1_PER_LANE=$2 python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" || exit 1
  echo "== warps $1 per-lane $2"; python tools/k1_stats.py cfg4 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', d['ms'])"; python tools/k1_stats.py cfg4 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('x8', d['ms'])"
done
python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)"
