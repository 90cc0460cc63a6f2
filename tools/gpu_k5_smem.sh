# K5 shared-memory pass (XM_K5=smem): parity (lifecycle, pipeline), timing vs
# the global-table kernel, ncu DRAM bytes of both.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "smem tests: $(XM_K5=smem timeout 900 python -m pytest tests/test_gpu_lifecycle.py tests/test_gpu_pipeline.py -x -q 2>&1 | grep -E 'passed|failed|Error' | tail -2)"
row() { python -c 'import sys,json; [print(json.loads(l).get("row","")[:12], {k:round(v,3) for k,v in json.loads(l).items() if k in ("ms","ms_without_wire","chain_instants_to_peaks_ms")}) for l in sys.stdin if l.strip().startswith("{")]' | tr '\n' ' '; }
for r in 1 2 3; do
  echo "global: $(timeout 300 python tools/bench_next.py lifecycle 2>/dev/null | row)"
  echo "smem:   $(XM_K5=smem timeout 300 python tools/bench_next.py lifecycle 2>/dev/null | row)"
done
mkdir -p gpurun_out/prof
XM_K5=smem timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_reconstruct python tools/bench_next.py lifecycle > gpurun_out/prof/ncu_k5smem.txt 2>&1
grep -E "k_reconstruct|dram__bytes|gpu__time" gpurun_out/prof/ncu_k5smem.txt | head -16
