python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_lifecycle.py -x -q 2>&1 | tail -1
timeout 900 python tools/bench_next.py lifecycle 2>&1 | grep '^{'
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_reconstruct -c 1 python tools/bench_next.py lifecycle 2>&1 | grep -E "dram__|gpu__time" | head
