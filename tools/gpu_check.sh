set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 600 python tools/lb_sweep.py ta091:1048576 ta021:1048576 ta051:1048576 ta111:262144 > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lb_kernel -s 3 -c 1 -o gpurun_out/prof_lb4 python bench.py --steps 1 --warmup 3 --no-bb --no-e2e --cpu-seconds 1 > gpurun_out/ncu4.log 2>&1
tail -1 gpurun_out/ncu4.log
