for b in 4 2 8; do echo "BEAM=$b"; FSP_BB_BEAM=$b timeout 300 python tools/bb_try.py ta091:2147483647:10 ta021:2147483647:10; done > gpurun_out/beam_sweep.txt 2>&1
for k in 12 20; do echo "K=$k BEAM=8"; FSP_BB_K=$k FSP_BB_BEAM=8 timeout 300 python tools/bb_try.py ta091:2147483647:10; done >> gpurun_out/beam_sweep.txt 2>&1
