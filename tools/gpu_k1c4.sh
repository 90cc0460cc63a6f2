python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_k1_paths.py -x -q 2>&1 | tail -2
XM_K1=t timeout 120 python tools/k1_stats.py cfg4 1
for cfg in "256 8 3 3" "256 8 2 4" "128 8 3 6"; do
  set -- $cfg
  XM_K1C_THREADS=$1 XM_K1C_PER=$2 XM_K1C_STAGES=$3 XM_K1C_CTAS_PER_SM=$4 python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "K1c threads=$1 per=$2 stages=$3 ctas=$4"; XM_K1=c timeout 120 python tools/k1_stats.py cfg4 1; XM_K1=c timeout 120 python tools/k1_stats.py cfg4 8
done
python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_scan_chunks -s 2 -c 1 -o gpurun_out/prof/k_scan_chunks9 env XM_K1=c python tools/k1_stats.py cfg4 1 > /dev/null 2>&1
