for w in 12 8; do for b in 2 3 4; do echo "WARPS=$w DBUF=$b"; FSP_LB_WARPS=$w FSP_LB_DBUF=$b timeout 300 python tools/lb_prof.py ta111:1048576; done; done > gpurun_out/sweep500.txt 2>&1
