timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 >> gpurun_out/pytest_gpu.txt
