timeout 900 python -m pytest tests/test_gpu_bb.py -x -q 2>&1 | tail -1
timeout 300 python tools/bb_try.py ta091:2147483647:10 ta051:2147483647:10 ta021:2147483647:10 ta005:2147483647:5
FSP_LB_PROF=1 timeout 120 python tools/bb_try.py ta091:2147483647:4 2>&1 | python tools/bb_prof.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 1200 --csv --log-file gpurun_out/launches_bb_r02b.csv python tools/bb_try.py ta091:2147483647:25 > /dev/null 2>&1; python tools/launch_shares.py gpurun_out/launches_bb_r02b.csv
