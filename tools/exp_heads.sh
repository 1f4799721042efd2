timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for cfg in "FSP_LB_SORT=1 FSP_LB_LANE_HEADS=1" "FSP_LB_SORT=1 FSP_LB_LANE_HEADS=0" "FSP_LB_SORT=0 FSP_LB_LANE_HEADS=1" "FSP_LB_SORT=0 FSP_LB_LANE_HEADS=0"; do echo "$cfg"; env $cfg timeout 300 python tools/lb_prof.py ta091:1048576 ta111:262144 ta051:1048576 ta021:1048576 ta001:1048576 2>&1 | cut -c1-125; done
