#!/bin/bash
# e2e event-input modes: parity of each mode, then the bench line's e2e numbers
set -e
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host_entry" 2>&1 | tail -2
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>gpurun_out/bench21.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('kernel', d['ms_per_step'], 'e2e', e['ms_per_step'], 'stream', e['stream_copy_ms_per_step'], e['results_equal_device_path'], e['api'][:90])"
done
