python tools/sanitize_run.py 2>&1 | tail -14
for t in memcheck racecheck initcheck; do
echo "== $t"; timeout 1500 compute-sanitizer --tool $t --print-limit 5 python tools/sanitize_run.py 2>&1 | grep -E "ERROR SUMMARY|Hazard|Invalid|Uninitialized|at void|at smc" | sort | uniq -c | head -10
done
echo "== synccheck"; timeout 1500 compute-sanitizer --tool synccheck --print-limit 5 python tools/sanitize_run.py --step-only 2>&1 | grep -E "ERROR SUMMARY|at void|Barrier" | sort | uniq -c | head -10
