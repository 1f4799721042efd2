for b in 2.0 4.0 8.0; do FSP_BB_BEAM=$b FSP_BB_CHILDREN=4194304 timeout 300 python tools/bb_try.py ta091:2147483647:30 ta111:2147483647:10 ta021:2147483647:10 2>&1 | sed "s/^/beam=$b /"; done
FSP_BB_BEAM=4.0 timeout 600 python -m pytest tests/test_gpu_bb.py -x -q 2>&1 | tail -1
