timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/sort_parity.log 2>&1; echo "rc=$?" >> gpurun_out/sort_parity.log
for so in 1 0; do echo "SORT=$so"; FSP_LB_SORT=$so timeout 300 python tools/lb_prof.py ta091:1048576 ta021:1048576 ta051:1048576 ta111:1048576 ta001:1048576; done 2>&1 | grep -v "^FSP" > gpurun_out/sort_prof.txt
