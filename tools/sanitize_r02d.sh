mkdir -p gpurun_out/san_r02d
for tool in memcheck synccheck; do timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_r02d/sanitize_$tool.txt 2>&1; echo "exit=$?" >> gpurun_out/san_r02d/sanitize_$tool.txt; done
FSP_LB_DBUF=0 timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_r02d/sanitize_racecheck_dbuf0.txt 2>&1; echo "exit=$?" >> gpurun_out/san_r02d/sanitize_racecheck_dbuf0.txt
