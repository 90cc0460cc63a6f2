XM_DEBUG=1 timeout 120 python tools/debug_run.py all > gpurun_out/debug_all.log 2>&1
tail -20 gpurun_out/debug_all.log
for k in H1a H1b H2a H3-early H3-late H4-late H5-two H6 H7 S251 S252 S260 S261 S262 S269 S270 P169 P654; do
  echo "== $k"; XM_DEBUG=1 timeout 60 python tools/debug_run.py $k 2>&1 | tail -2
done
