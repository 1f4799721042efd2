timeout 900 python -m pytest tests/test_gpu_bb.py -x -q 2>&1 | tail -3
for F in 1 0; do for K in 8 32; do FSP_BB_FAMILY=$F FSP_BB_K=$K timeout 300 python tools/bb_try.py ta001:2147483647:30 ta003:2147483647:30 ta021:2147483647:10 ta051:2147483647:10 ta091:2147483647:10 2>&1 | sed "s/^/F=$F K=$K /" | cut -c1-230; done; done
