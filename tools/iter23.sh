#!/bin/bash
# hybrid host input: parity of every mode, then e2e per mode and per first-wave size
set -e
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed or host_entry" 2>&1 | tail -2
python tools/e2e_probe.py
for nd in 1000 2072 3000 4000; do
  for m in hybrid; do
    XM_DIRECT_TRACES=$nd XM_E2E_MODES="$m" python tools/e2e_modes.py
  done
done
python tools/e2e_modes.py direct stream copy
