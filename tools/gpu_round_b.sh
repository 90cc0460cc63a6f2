# K2 A/B (tree vs ab_tmp variants), GPU suite, K1t/K1c geometry sweeps.
mkdir -p gpurun_out
bash tools/ab_k2.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for cfg in "4 8" "4 16" "8 8" "8 4" "2 16"; do
  set -- $cfg
  XM_K1_WARPS=$1 XM_K1_PER_LANE=$2 python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "K1t warps=$1 per_lane=$2"; XM_K1=t timeout 120 python tools/k1_stats.py cfg4 1
done
for cfg in "128 8 2 8" "128 8 3 6" "128 16 2 4" "256 8 2 4"; do
  set -- $cfg
  XM_K1C_THREADS=$1 XM_K1C_PER=$2 XM_K1C_STAGES=$3 XM_K1C_CTAS_PER_SM=$4 python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "K1c threads=$1 per=$2 stages=$3 ctas=$4"; XM_K1=c timeout 120 python tools/k1_stats.py cfg4 1
done
python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
