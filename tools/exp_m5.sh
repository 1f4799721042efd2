timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config_pools or machine_counts or boundary or job_pairs or 20x5 or fixed_depths or degenerate or strides or malformed or duplicates" > gpurun_out/m5_parity.log 2>&1; echo "rc=$?" >> gpurun_out/m5_parity.log
timeout 600 python -m pytest tests/test_gpu_bb.py -x -q > gpurun_out/m5_bb.log 2>&1; echo "rc=$?" >> gpurun_out/m5_bb.log
for jp in 1 0; do echo "JP=$jp"; FSP_LB_JP=$jp timeout 300 python tools/lb_prof.py ta001:1048576 ta001:65536; done > gpurun_out/m5_prof.txt 2>&1
