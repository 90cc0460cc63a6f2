XM_DEBUG=1 timeout 60 python tools/debug_run.py H1a 2>&1 | head -60
