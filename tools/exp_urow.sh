for pad in 1 0; do echo "PAD=$pad"; FSP_LB_UROW_PAD=$pad timeout 300 python tools/lb_prof.py ta091:1048576 ta021:1048576 ta051:1048576; done > gpurun_out/urow_prof.txt 2>&1
FSP_LB_UROW_PAD=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config_pools or full_size_200 or fixed_depths" > gpurun_out/urow_parity.log 2>&1; echo "rc=$?" >> gpurun_out/urow_parity.log
