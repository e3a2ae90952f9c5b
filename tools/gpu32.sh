for tool in synccheck racecheck memcheck; do
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 10 python tools/sanitize_run.py > gpurun_out/san_$tool.txt 2>&1; echo "$tool rc=$?"; grep -m3 -E "Error|error" gpurun_out/san_$tool.txt; tail -2 gpurun_out/san_$tool.txt
done
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
