# NEXT-row measurements + ncu of their kernels (one GPU)
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python tools/bench_next.py lifecycle metrics k4 > gpurun_out/bench_next.jsonl 2> gpurun_out/bench_next.err
cat gpurun_out/bench_next.jsonl; tail -3 gpurun_out/bench_next.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_reconstruct -s 1 -c 1 -o gpurun_out/prof/k_reconstruct python tools/bench_next.py lifecycle > gpurun_out/prof/ncu_k5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_expand -s 1 -c 1 -o gpurun_out/prof/k_expand python tools/bench_next.py k4 > gpurun_out/prof/ncu_k4.log 2>&1
ls gpurun_out/prof
