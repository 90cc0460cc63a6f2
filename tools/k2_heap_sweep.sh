# K2 time vs the shared-memory heap size (smem_per_warp x 14 warps): how much
# does the number of resident traces matter?
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for spw in 0 14336 12288 10240 8192; do SPW=$spw timeout 120 python tools/k2_stats.py cfg4 14; done
for spw in 0 12288; do SPW=$spw timeout 120 python tools/k2_stats.py cfg4 12,16; done
