# A/B of K1t runtime settings on config 4 (same library, environment variants):
# usage: bash tools/ab_k1_env.sh "NAME:ENV=VAL ..." ...
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_k1_paths.py -x -q 2>&1 | tail -1
for r in 1 2 3; do
  echo "tree: $(XM_K1=t timeout 120 python tools/k1_stats.py ${K1_WL:-cfg4} ${K1_REP:-1} | cut -c1-150)"
  for v in "$@"; do
    echo "${v%%:*}: $(env XM_K1=t ${v#*:} timeout 120 python tools/k1_stats.py ${K1_WL:-cfg4} ${K1_REP:-1} | cut -c1-150)"
  done
done
