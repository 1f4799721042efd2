for w in 14 12 8; do FSP_LB_PAD=1 FSP_LB_NPL=4 SWEEP_WARPS=$w timeout 600 python tools/lb_sweep.py ta091:1048576 2>&1 | tail -1; done
FSP_LB_PAD=1 timeout 600 python tools/lb_sweep.py ta091:1048576 2>&1 | tail -1
