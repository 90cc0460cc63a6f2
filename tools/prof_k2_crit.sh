# ncu source-level captures of K2: the longest config-4 trace alone (its serial
# chain) and the whole config-4 launch.
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/k2_subset.py resnet152/adamw/pos1/b600/r0 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 1 -c 1 -o gpurun_out/prof/k_replay_crit python tools/k2_subset.py resnet152/adamw/pos1/b600/r0 1 > gpurun_out/prof/ncu_crit.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 3 -c 1 -o gpurun_out/prof/k_replay_src python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-k1 > gpurun_out/prof/ncu_k2src.log 2>&1
ls -la gpurun_out/prof
