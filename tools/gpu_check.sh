set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
FSP_LB_NPL=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5 >> gpurun_out/pytest_gpu.txt
FSP_LB_NPL=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5 >> gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
SWEEP_NPL=0 SWEEP_WARPS=0 timeout 600 python tools/lb_sweep.py ta091:1048576 ta021:1048576 ta051:1048576 ta001:1048576 ta111:262144 > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
