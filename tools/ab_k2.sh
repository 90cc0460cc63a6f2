# A/B timing of K2 on one box: the tree's replay.cu vs ab_tmp/replay_*.cu
# variants and vs ab_tmp/variants.txt lines ("name WPC ENV=VAL ..." = the tree
# built with those macros, timed at WPC warps per CTA), each a separately named
# library, timed alternately on config 4.
set -e
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
names=()
for f in ab_tmp/replay_*.cu; do
  [ -e "$f" ] || continue
  t=$(basename $f .cu); XM_BUILD_TAG=$t XM_REPLAY_SRC=$f python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  names+=("$t:14")
done
if [ -f ab_tmp/variants.txt ]; then
  while read -r name wpc envs; do
    [ -z "$name" ] && continue
    env XM_BUILD_TAG=$name $envs python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
    names+=("$name:$wpc")
  done < ab_tmp/variants.txt
fi
for r in 1 2 3; do
  echo "tree: $(timeout 120 python tools/k2_stats.py cfg4 14)"
  for nw in "${names[@]}"; do
    t=${nw%%:*}; wpc=${nw##*:}
    echo "$t: $(XM_LIB=paper_2510_21048_b200/libxmem_$t.so timeout 120 python tools/k2_stats.py cfg4 $wpc)"
  done
done
