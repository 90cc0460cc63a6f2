for fd in 2 4 8 16; do
  XM_F_INIT_DIV=$fd python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" || exit 1
  echo "== F init n_ids/$fd"; python tools/k2_stats.py cfg4 14,15
done
python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)"
