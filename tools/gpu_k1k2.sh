# K1c tuning sweep + the full GPU suite (K2 pool-partitioned free list).
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
XM_K1=t timeout 120 python tools/k1_stats.py cfg4 1
for cfg in "8 3 3" "8 4 2" "16 2 2" "8 2 4" "16 3 1"; do
  set -- $cfg
  XM_K1C_PER=$1 XM_K1C_STAGES=$2 XM_K1C_CTAS_PER_SM=$3 python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "cfg per=$1 stages=$2 ctas=$3"; XM_K1=c timeout 120 python tools/k1_stats.py cfg4 1; XM_K1=c timeout 120 python tools/k1_stats.py cfg4 8
done
python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
timeout 300 python tools/k2_stats.py cfg4 14
