for c in lr lrinp c2inp ssminp; do
timeout 600 compute-sanitizer --tool synccheck --print-limit 2 python tools/sync_probe2.py $c 2>&1 | grep -E "^[a-z]|ERROR SUMMARY|at void" | head -4
done
