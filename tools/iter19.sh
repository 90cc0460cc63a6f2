for nap in 16384 4096 1024; do
  XM_MAX_NAP=$nap python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)" || exit 1
  echo "== max nap $nap"; python tools/k2_stats.py cfg4 14,14
done
python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)"
