timeout 900 python -m pytest tests/test_gpu_bb.py -x -q 2>&1 | tail -1
for r in smem global; do FSP_BB_RECS=$r timeout 300 python tools/bb_try.py ta091:2147483647:10 2>&1 | sed "s/^/recs=$r /"; FSP_BB_RECS=$r FSP_LB_PROF=1 timeout 120 python tools/bb_try.py ta091:2147483647:4 2>&1 | python tools/bb_prof.py; done
FSP_BB_RECS=global timeout 900 python -m pytest tests/test_gpu_bb.py -x -q -k "child_pool or taillard" 2>&1 | tail -1
timeout 300 python tools/bb_try.py ta051:2147483647:10 ta021:2147483647:10 ta005:2147483647:5
