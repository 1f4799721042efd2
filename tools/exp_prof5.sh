for sk in 0 1 4 8; do echo "SKIP=$sk"; FSP_LB_DEBUG_SKIP=$sk timeout 300 python tools/lb_prof.py ta091:1048576; done > gpurun_out/prof5.txt 2>&1
