# bench line, per-config roofline sweep, ncu launch list + full capture of the bench kernel
timeout 900 python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err
rm -f gpurun_out/r02_sweep2.jsonl
for c in ta001 ta021 ta051 ta111; do timeout 300 python bench.py --config $c --no-bb --no-e2e --cpu-seconds 3 --steps 20 >> gpurun_out/r02_sweep2.jsonl 2>>gpurun_out/r02_sweep2.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02.csv python bench.py --steps 5 --warmup 3 --no-bb --no-e2e --cpu-seconds 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lb_kernel -s 3 -c 1 -o gpurun_out/lb_r02 python bench.py --steps 2 --warmup 3 --no-e2e --no-bb --cpu-seconds 1 > gpurun_out/ncu_lb_r02.log 2>&1
python tools/ncu_summary.py gpurun_out/lb_r02.ncu-rep > gpurun_out/lb_kernel_r02_ncu_summary.json 2>&1
