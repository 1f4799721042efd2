# source-level ncu of the B&B expand kernel and the B&B bounding kernel (one launch each, mid-search)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:expand_kernel -s 900 -c 1 -o gpurun_out/expand_r02b python tools/bb_try.py ta091:2147483647:60 > gpurun_out/ncu_expand.log 2>&1
python tools/ncu_summary.py gpurun_out/expand_r02b.ncu-rep > gpurun_out/expand_r02b_ncu_summary.json 2>&1
ncu -i gpurun_out/expand_r02b.ncu-rep --page source --csv > gpurun_out/expand_r02b_source.csv 2>/dev/null
