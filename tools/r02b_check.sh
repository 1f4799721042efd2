# session re-entry check: GPU tests, smoke, bench line
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02b_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
