timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lb_kernel -s 3 -c 1 -o gpurun_out/prof_lb6 python bench.py --steps 1 --warmup 3 --no-bb --no-e2e --cpu-seconds 1 > gpurun_out/ncu6.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-bb --no-e2e --cpu-seconds 1 > gpurun_out/ncu_launch_bench.log 2>&1
