for pg in 512 256 1024; do
  XM_PAGE=$pg python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" || exit 1
  echo "== page $pg"; python tools/k2_stats.py cfg4 14,15,16
done
python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)"
XM_PAGE=256 python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)"
