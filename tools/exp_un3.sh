for v in main sp2 sp4; do echo "VARIANT=$v"; if [ $v = main ]; then V=; else V=$v; fi; FSP_LIB_VARIANT=$V timeout 300 python tools/bb_try.py ta091:2147483647:10 ta021:2147483647:10; done > gpurun_out/un3_bb.txt 2>&1
timeout 300 python tools/lb_prof.py ta091:1048576 ta021:1048576 ta051:1048576 ta111:1048576 ta001:1048576 2>&1 | grep -v "^FSP" > gpurun_out/un3_prof.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bb.py -x -q > gpurun_out/un3_parity.log 2>&1; echo "rc=$?" >> gpurun_out/un3_parity.log
