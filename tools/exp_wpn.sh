timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "warp_per_node or 500x20" > gpurun_out/wpn_parity.log 2>&1; echo "rc=$?" >> gpurun_out/wpn_parity.log
echo "# mapping A/B: thread per node (product) vs warp per node (FSP_LB_MAPPING=warp)" > gpurun_out/wpn_ab.txt
for mp in thread warp; do echo "## $mp" >> gpurun_out/wpn_ab.txt; FSP_LB_MAPPING=$mp timeout 600 python tools/lb_prof.py ta001:1048576 ta021:1048576 ta051:1048576 ta091:1048576 ta111:262144 2>&1 | grep -v "^FSP" >> gpurun_out/wpn_ab.txt; done
