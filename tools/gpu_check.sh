set -x
timeout 900 python -m pytest tests/test_gpu_bb.py -x -q 2>&1 | tail -8
timeout 600 python tools/bb_try.py ta091:2147483647:20 ta051:2147483647:15 ta021:2147483647:15 ta002:2147483647:20 > gpurun_out/bb_try.txt 2>&1; cat gpurun_out/bb_try.txt
for k in 4 16 64; do FSP_BB_K=$k timeout 600 python tools/bb_try.py ta091:2147483647:15 2>&1 | sed "s/^/K=$k /"; done
