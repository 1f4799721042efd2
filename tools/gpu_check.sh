timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bb.py -x -q 2>&1 | tail -2
for k in 8 16; do FSP_BB_K=$k timeout 600 python tools/bb_try.py ta091:2147483647:15 2>&1 | sed "s/^/npl2 K=$k /" | cut -c1-60,200-300; done
FSP_BB_NPL=4 timeout 600 python tools/bb_try.py ta091:2147483647:15 2>&1 | sed "s/^/npl4 K=8 /" | cut -c1-60,200-300
timeout 600 python tools/bb_try.py ta051:2147483647:15 ta021:2147483647:15 2>&1 | cut -c1-60,200-300
