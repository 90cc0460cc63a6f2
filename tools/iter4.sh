python -c "import __graft_entry__ as g; g.build()" || exit 1
XM_TIMING=1 python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)"
python tools/k2_timing.py 12 2>&1 | tail -12
ls -la gpurun_out/
