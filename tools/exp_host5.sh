timeout 900 python tools/exp_host.py "" "FSP_HOST_TAIL=2" "FSP_HOST_TAIL=1" "FSP_HOST_TAIL=2,FSP_GATHER_SMS=10" > gpurun_out/host5_sweep.txt 2>&1
