for k in 8 6 12 16; do echo "K=$k"; FSP_BB_K=$k timeout 300 python tools/bb_try.py ta091:2147483647:10 ta021:2147483647:10 ta111:2147483647:10; done > gpurun_out/k_sweep.txt 2>&1
