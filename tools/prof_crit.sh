# Critical-path analysis of K2: per-trace timing (XM_TIMING build) on config 4,
# the longest trace replayed alone, and an ncu source-level capture of it.
set -x
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()"
XM_TIMING=1 python -c "from paper_2510_21048_b200 import _build; _build.build(force=True)"
python tools/k2_timing.py 12 > gpurun_out/prof/k2_timing.log 2>&1; cat gpurun_out/prof/k2_timing.log
python tools/k2_subset.py resnet152/adamw/pos1/b600/r0 1
python tools/k2_subset.py resnet152/adamw 12
python tools/k2_subset.py llama3.2 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 1 -c 1 -o gpurun_out/prof/k_replay_crit python tools/k2_subset.py resnet152/adamw/pos1/b600/r0 1 > /dev/null 2>&1
ls gpurun_out/prof/
