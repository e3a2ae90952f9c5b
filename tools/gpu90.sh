timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 python tools/sanitize_run.py --step-only > gpurun_out/racecheck_step.log 2>&1; echo rc=$?
grep -E "ERROR SUMMARY|Hazard|RACECHECK SUMMARY" gpurun_out/racecheck_step.log | sort | uniq -c | head; tail -4 gpurun_out/racecheck_step.log
