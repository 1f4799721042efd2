timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
