timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config_pools or kcache or full_size or job_pairs or machine_counts" > gpurun_out/kc3_parity.log 2>&1; echo "rc=$?" >> gpurun_out/kc3_parity.log
timeout 300 python tools/lb_prof.py ta091:1048576 ta021:1048576 ta051:1048576 ta111:1048576 ta001:1048576 2>&1 | grep -v "^FSP" > gpurun_out/kc3_prof.txt
