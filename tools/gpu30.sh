for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py 2>&1 | grep -vE "^(crbd|clads2|seir|geometric|virtual|resampler)" | tail -15
  echo "rc=${PIPESTATUS[0]}"
done
