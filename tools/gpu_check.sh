set -x
timeout 600 python tools/bb_try.py ta091:2147483647:20 ta051:2147483647:20 ta021:2147483647:20 > gpurun_out/bb_try.txt 2>&1; cat gpurun_out/bb_try.txt
FSP_BB_STACK=200000 timeout 600 python tools/bb_try.py ta091:2147483647:10 > gpurun_out/bb_try2.txt 2>&1; cat gpurun_out/bb_try2.txt
