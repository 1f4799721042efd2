set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 600 python tools/bb_try.py ta002:2147483647:30 ta001:1278:60 ta001:2147483647:30 ta091:2147483647:20 > gpurun_out/bb_try.txt 2>&1; cat gpurun_out/bb_try.txt
