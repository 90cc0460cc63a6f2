# A/B timing of K2 on one box: ab_tmp/replay_*.cu variants vs the tree's
# replay.cu, built as separate libraries and timed alternately (config 4).
set -e
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for f in ab_tmp/replay_*.cu; do
  t=$(basename $f .cu); XM_BUILD_TAG=$t XM_REPLAY_SRC=$f python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
done
for r in 1 2 3; do
  echo "tree: $(timeout 120 python tools/k2_stats.py cfg4 14)"
  for f in ab_tmp/replay_*.cu; do
    t=$(basename $f .cu); echo "$t: $(XM_LIB=paper_2510_21048_b200/libxmem_$t.so timeout 120 python tools/k2_stats.py cfg4 14)"
  done
done
