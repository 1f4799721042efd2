timeout 600 python tools/bb_try.py ta091:2147483647:15 ta051:2147483647:10 ta021:2147483647:10 ta002:2147483647:10 > gpurun_out/bbt.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bb.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2 >> gpurun_out/bbt.txt
