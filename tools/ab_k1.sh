# A/B timing of K1t on config 4: the tree vs ab_tmp/scan_old.cu and the build
# variants listed in ab_tmp/k1_variants.txt ("name ENV=VAL ..."), each a
# separately named library, timed alternately; the K1 parity tests run
# against every variant first.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
L=paper_2510_21048_b200
names=()
if [ -f ab_tmp/scan_old.cu ]; then
  XM_BUILD_TAG=k1old XM_SCAN_SRC=ab_tmp/scan_old.cu python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  names+=(k1old)
fi
if [ -f ab_tmp/k1_variants.txt ]; then
  while read -r name envs; do
    [ -z "$name" ] && continue
    env XM_BUILD_TAG=$name $envs python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
    names+=("$name")
  done < ab_tmp/k1_variants.txt
fi
echo "tree: $(timeout 600 python -m pytest tests/test_gpu_k1_paths.py -x -q 2>&1 | tail -1)"
for t in "${names[@]}"; do echo "$t: $(XM_LIB=$L/libxmem_$t.so timeout 600 python -m pytest tests/test_gpu_k1_paths.py -x -q 2>&1 | tail -1)"; done
for r in 1 2 3; do
  echo "tree: $(XM_K1=t timeout 120 python tools/k1_stats.py ${K1_WL:-cfg4} 1 | cut -c1-140)"
  for t in "${names[@]}"; do echo "$t: $(XM_K1=t XM_LIB=$L/libxmem_$t.so timeout 120 python tools/k1_stats.py ${K1_WL:-cfg4} 1 | cut -c1-140)"; done
done
