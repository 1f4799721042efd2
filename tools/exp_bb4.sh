timeout 900 python -m pytest tests/test_gpu_bb.py tests/test_dist.py -x -q -m gpu > gpurun_out/bb4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bb4_tests.log
timeout 600 python tools/bb_try.py ta091:2147483647:10 ta021:2147483647:10 ta051:2147483647:10 ta111:2147483647:10 ta001:2147483647:10 > gpurun_out/bb4.txt 2>&1
