./tools/ubench/ipipe > gpurun_out/ipipe_r02b.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config_pools or machine_counts or boundary or job_pairs or full_size_200 or fixed_depths or degenerate" > gpurun_out/jp2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/jp2_parity.log
timeout 300 python tools/lb_prof.py ta091:1048576 ta021:1048576 ta051:1048576 ta111:1048576 ta001:1048576 > gpurun_out/jp2_prof.txt 2>&1
