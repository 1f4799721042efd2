timeout 1500 python bench.py --table2 > gpurun_out/table2_r02e.jsonl 2> gpurun_out/table2_r02e.err
