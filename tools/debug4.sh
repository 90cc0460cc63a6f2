SPW=16384 WPC=1 XM_DEBUG=1 timeout 120 python tools/debug_run.py frag2 2>&1 | tail -2 | cut -c1-300
SPW=16384 WPC=1 timeout 120 python tools/debug_run.py frag2 2>&1 | tail -1 | cut -c1-300
SPW=16384 WPC=1 timeout 120 python tools/debug_run.py frag 2>&1 | tail -1 | cut -c1-300
timeout 120 python tools/debug_run.py frag2 2>&1 | tail -1 | cut -c1-300
SPW=16384 WPC=1 timeout 300 compute-sanitizer --print-limit 3 python tools/debug_run.py frag2 2>&1 | grep -v "Host Frame" | head -30
