timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 python tools/sanitize_run.py > gpurun_out/racecheck.log 2>&1; echo rc=$?
grep -E "ERROR SUMMARY|Hazard|RACECHECK SUMMARY" gpurun_out/racecheck.log | sort | uniq -c | head; tail -5 gpurun_out/racecheck.log
