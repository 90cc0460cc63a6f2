for k in H1a H1b H1c H1d H2a H2b H3-early H3-late H4-late H4-early H5-two H5-one H6 H7 S251 S252 S260 S261 S262 S269 S270 P169 P654 P654-10MiB; do
  echo "== $k"; XM_DEBUG=1 timeout 60 python tools/debug_run.py $k 2>&1 | grep -v "^  " | tail -1 | cut -c1-200
done
