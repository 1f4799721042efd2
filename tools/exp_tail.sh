for t in 1 0; do echo "TAIL=$t"; FSP_LB_TAIL=$t python tools/lb_prof.py ta091:1048576 ta111:262144 ta051:1048576 ta021:1048576 ta001:1048576 ta091:600000 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
