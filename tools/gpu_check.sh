timeout 600 python tools/bb_try.py ta091:2147483647:15 > gpurun_out/bbt.txt 2>&1
timeout 600 python tools/lb_sweep.py ta091:1048576 ta021:1048576 ta051:1048576 >> gpurun_out/bbt.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bb.py -x -q 2>&1 | tail -2 >> gpurun_out/bbt.txt
