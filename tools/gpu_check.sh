set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-bb --no-e2e --cpu-seconds 1 > gpurun_out/ncu_launch_bench.log 2>&1
tail -2 gpurun_out/ncu_launch_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 600 --csv --log-file gpurun_out/launches_bb.csv python tools/bb_try.py ta091:2147483647:20 > gpurun_out/ncu_launch_bb.log 2>&1
tail -2 gpurun_out/ncu_launch_bb.log
