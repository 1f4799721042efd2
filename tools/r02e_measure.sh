timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/r02e_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r02e_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
