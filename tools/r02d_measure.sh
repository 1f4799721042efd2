# round-2 end: full GPU suite, smoke, bench line, launch list, ncu of the bench kernel
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/r02d_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02d.csv python bench.py --steps 5 --warmup 3 --no-bb --no-e2e --no-configs --cpu-seconds 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lb_kernel -s 3 -c 1 -o gpurun_out/lb_r02d python bench.py --steps 2 --warmup 3 --no-e2e --no-bb --no-configs --cpu-seconds 1 > gpurun_out/ncu_lb_r02d.log 2>&1
python tools/ncu_summary.py gpurun_out/lb_r02d.ncu-rep > gpurun_out/lb_kernel_r02d_ncu_summary.json 2>&1
