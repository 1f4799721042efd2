timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bb.py -x -q 2>&1 | tail -2
timeout 300 python tools/lb_prof.py ta091:1048576 ta111:262144 ta051:1048576 ta021:1048576 ta001:1048576 2>&1 | cut -c1-125
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none -k regex:lb_kernel -s 3 -c 1 python tools/lb_prof.py ta091:1048576 2>&1 | grep -E "duration|bytes|pct|ratio"
