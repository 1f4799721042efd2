timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host_api" > gpurun_out/host2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/host2_parity.log
timeout 900 python tools/exp_host.py "" "FSP_HOST_NOTAIL=1" "FSP_GATHER_SMS=10" "FSP_GATHER_SMS=12" "FSP_GATHER_SMS=6" "FSP_GATHER_ONLY=1" > gpurun_out/host2_sweep.txt 2>&1
