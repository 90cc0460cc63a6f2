# ncu source-level capture of k_replay on config 4 (SASS inst-executed and stall
# sampling per line), plus the config-1 single-trace replay (latency view).
set -x
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 3 -c 1 -o gpurun_out/prof/k_replay_src python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_k2src.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 3 -c 1 -o gpurun_out/prof/k_replay_cfg1 python bench.py --workload cfg1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_k2cfg1.log 2>&1
ls -la gpurun_out/prof
