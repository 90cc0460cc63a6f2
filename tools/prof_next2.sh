mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python tools/bench_next.py orchestrate > gpurun_out/bench_next2.jsonl 2> gpurun_out/bench_next2.err
cat gpurun_out/bench_next2.jsonl; tail -3 gpurun_out/bench_next2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_orchestrate -s 1 -c 1 -o gpurun_out/prof/k_orchestrate python tools/bench_next.py orchestrate > gpurun_out/prof/ncu_k6.log 2>&1
ls gpurun_out/prof
