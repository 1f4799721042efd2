set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 600 python tools/lb_sweep.py ta091:1048576 ta021:1048576 ta051:1048576 ta111:262144 ta001:1048576 > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-bb > gpurun_out/bench1.json 2> gpurun_out/bench1.err
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lb_kernel -s 3 -c 1 -o gpurun_out/prof_lb2 python bench.py --steps 1 --warmup 3 --no-bb --no-e2e --cpu-seconds 1 > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
