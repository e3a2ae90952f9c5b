mkdir -p gpurun_out/san
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py --step-only > gpurun_out/san/synccheck.log 2>&1; echo "synccheck: $(grep -E "ERROR SUMMARY" gpurun_out/san/synccheck.log | tail -1)"
grep -E "^[a-z]|at void" gpurun_out/san/synccheck.log | sort | uniq -c | sort -rn | head -5
