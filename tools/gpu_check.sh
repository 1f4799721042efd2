SWEEP_NPL=0 SWEEP_WARPS=0 timeout 600 python tools/lb_sweep.py ta091:1048576 ta051:1048576 ta021:1048576 ta001:1048576 ta111:262144 2>&1 | grep cfg > gpurun_out/sweep_grid.txt
timeout 600 python tools/bb_try.py ta091:2147483647:15 ta051:2147483647:10 ta021:2147483647:10 >> gpurun_out/sweep_grid.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bb.py -x -q 2>&1 | tail -2 >> gpurun_out/sweep_grid.txt
