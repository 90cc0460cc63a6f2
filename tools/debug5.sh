XM_DEBUG=1 timeout 120 python tools/debug_run.py frag2 > gpurun_out/dbg5.log 2>&1
grep -v "^  \|Traceback\|File\|raise\|_check\|h, s\|h, summ" gpurun_out/dbg5.log | head -30 | cut -c1-250
