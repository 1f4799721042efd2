timeout 900 python -m pytest tests/test_gpu_bb.py tests/test_dist.py -x -q -m gpu --timeout=300 > gpurun_out/k2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k2_tests.log
timeout 300 python tools/bb_try.py ta001:2147483647:30 ta002:2147483647:30 ta003:2147483647:60 ta004:2147483647:60 > gpurun_out/k2_solves.txt 2>&1
