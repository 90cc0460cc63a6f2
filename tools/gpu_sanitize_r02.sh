# round 2: the heap hand-off stress test, then every kernel path under
# compute-sanitizer (memcheck, synccheck, racecheck).
mkdir -p gpurun_out/sanitizer
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heap_page or launch_geom or fragmentation" 2>&1 | tail -2
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/sanitizer/r02_$tool.txt 2>&1
  echo "== $tool: exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize run done" gpurun_out/sanitizer/r02_$tool.txt | head -4
done
