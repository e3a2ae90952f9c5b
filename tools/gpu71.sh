timeout 1500 compute-sanitizer --tool synccheck --print-limit 5 python tools/sanitize_run.py --step-only 2>&1 | grep -E "^[a-z]|ERROR SUMMARY|at void" | sort | uniq -c | head -20
