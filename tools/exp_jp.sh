# job-pair heads: parity, A/B timing and phase split, integer-pipe ubench
./tools/ubench/ipipe > gpurun_out/ipipe_r02b.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/jp_parity.log 2>&1; echo "rc=$?" >> gpurun_out/jp_parity.log
for jp in 1 0; do
  FSP_LB_JP=$jp timeout 300 python tools/lb_prof.py ta091:1048576 ta021:1048576 ta051:1048576 ta111:1048576 > gpurun_out/jp_prof_$jp.txt 2>&1
done
