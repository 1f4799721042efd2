timeout 900 python -m pytest tests/test_gpu_bb.py -x -q 2>&1 | tail -1
for l in 1 0; do FSP_BB_LAZY=$l timeout 300 python tools/bb_try.py ta091:2147483647:10 ta111:2147483647:10 2>&1 | sed "s/^/lazy=$l /"; done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -s 8000 -c 1200 --csv --log-file gpurun_out/launches_bb_r02d.csv python tools/bb_try.py ta091:2147483647:30 > /dev/null 2>&1; python tools/launch_shares.py gpurun_out/launches_bb_r02d.csv
