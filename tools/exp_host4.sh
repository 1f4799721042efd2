timeout 900 python tools/exp_host.py "" "FSP_HOST_TAIL=1" "FSP_HOST_TAIL=1,FSP_HOST_NORAMP=1" "FSP_HOST_LASTSPLIT=1" > gpurun_out/host4_sweep.txt 2>&1
