timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout=300 > gpurun_out/p8b_parity.log 2>&1; echo "rc=$?" >> gpurun_out/p8b_parity.log
for e in "X=1" "FSP_LB_PTM8=0"; do echo "ENV $e"; env $e timeout 300 python tools/lb_prof.py ta091:1048576 ta021:1048576 ta051:1048576 ta111:1048576 ta001:1048576; done 2>&1 | grep -v "^FSP" > gpurun_out/p8b_prof.txt
