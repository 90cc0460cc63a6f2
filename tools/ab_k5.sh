# A/B of K5 (k_reconstruct): the tree vs ab_tmp/lifecycle_old.cu, parity
# tests on both, then bench_next's lifecycle and pipeline rows alternately.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
XM_BUILD_TAG=k5old XM_LIFECYCLE_SRC=ab_tmp/lifecycle_old.cu python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
L=paper_2510_21048_b200
echo "tree: $(timeout 900 python -m pytest tests/test_gpu_lifecycle.py tests/test_gpu_pipeline.py -x -q 2>&1 | grep -E 'passed|failed' | tail -1)"
echo "tree k5 loader: $(XM_LOADER=k5 timeout 900 python -m pytest tests/test_gpu_raw.py -x -q 2>&1 | grep -E 'passed|failed' | tail -1)"
for r in 1 2 3; do
  echo "tree: $(timeout 300 python tools/bench_next.py lifecycle pipeline 2>/dev/null | python -c 'import sys,json; [print(json.loads(l).get("row","")[:30], {k:v for k,v in json.loads(l).items() if k.endswith("ms") or k=="ms_per_step"}) for l in sys.stdin if l.strip().startswith("{")]' | tr '\n' ' ')"
  echo "old:  $(XM_LIB=$L/libxmem_k5old.so timeout 300 python tools/bench_next.py lifecycle pipeline 2>/dev/null | python -c 'import sys,json; [print(json.loads(l).get("row","")[:30], {k:v for k,v in json.loads(l).items() if k.endswith("ms") or k=="ms_per_step"}) for l in sys.stdin if l.strip().startswith("{")]' | tr '\n' ' ')"
done
