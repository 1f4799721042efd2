timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config_pools or machine_counts or boundary or job_pairs or full_size_200 or fixed_depths" > gpurun_out/jp3_parity.log 2>&1; echo "rc=$?" >> gpurun_out/jp3_parity.log
for sk in 0 4 8 12 1; do echo "SKIP=$sk"; FSP_LB_DEBUG_SKIP=$sk timeout 300 python tools/lb_prof.py ta091:1048576 ta021:1048576; done > gpurun_out/jp3_prof.txt 2>&1
