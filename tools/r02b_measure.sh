# round-2b measurement: bench line, launch list, ncu full of the bench kernel and of the A/B kernel
timeout 900 python bench.py > gpurun_out/r02b_bench2.json 2> gpurun_out/r02b_bench2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02b.csv python bench.py --steps 5 --warmup 3 --no-bb --no-e2e --no-configs --cpu-seconds 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lb_kernel -s 3 -c 1 -o gpurun_out/lb_r02b python bench.py --steps 2 --warmup 3 --no-e2e --no-bb --no-configs --cpu-seconds 1 > gpurun_out/ncu_lb_r02b.log 2>&1
python tools/ncu_summary.py gpurun_out/lb_r02b.ncu-rep > gpurun_out/lb_kernel_r02b_ncu_summary.json 2>&1
FSP_LB_MAPPING=warp timeout 900 ncu --set full --clock-control none -k regex:lb_wpn -s 1 -c 1 -o gpurun_out/wpn_r02b python tools/lb_prof.py ta091:262144 > gpurun_out/ncu_wpn_r02b.log 2>&1
python tools/ncu_summary.py gpurun_out/wpn_r02b.ncu-rep > gpurun_out/wpn_r02b_ncu_summary.json 2>&1
