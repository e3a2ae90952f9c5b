for c in a b c d e; do
timeout 600 compute-sanitizer --tool synccheck --print-limit 2 python tools/sync_probe.py $c 2>&1 | grep -E "^[a-e] |ERROR SUMMARY|at void" | head -3
done
