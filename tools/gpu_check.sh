for v in 1 0; do FSP_LB_VECROWS=$v SWEEP_NPL=0 SWEEP_WARPS=0 timeout 600 python tools/lb_sweep.py ta051:1048576 2>&1 | grep cfg | sed "s/^/vec=$v /"; done
for v in 1 0; do FSP_LB_VECROWS=$v timeout 600 python tools/bb_try.py ta051:2147483647:10 ta021:2147483647:10 2>&1 | sed "s/^/vec=$v /" | cut -c1-70,200-320; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bb.py -x -q 2>&1 | tail -1
