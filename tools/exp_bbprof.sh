FSP_LB_PROF=1 timeout 300 python tools/bb_try.py ta091:2147483647:5 2>&1 | python tools/bb_prof.py > gpurun_out/bbprof.txt
FSP_LB_PROF=1 timeout 300 python tools/bb_try.py ta021:2147483647:5 2>&1 | python tools/bb_prof.py >> gpurun_out/bbprof.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bb_r02c.csv -c 1500 python tools/bb_try.py ta091:2147483647:3 > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/launches_bb_r02c.csv >> gpurun_out/bbprof.txt
