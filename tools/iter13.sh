for div in 16 24 64; do
  XM_HEAP_RESERVE_DIV=$div python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" || exit 1
  echo "== reserve 1/$div"; python tools/k2_stats.py cfg4 13,14,15
done
python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)"
