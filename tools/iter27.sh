#!/bin/bash
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "host_" 2>&1 | tail -2
python tools/e2e_modes.py direct stream
