mkdir -p gpurun_out/san
for tool in memcheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san/$tool.log | tail -2)"
done
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py --step-only > gpurun_out/san/synccheck.log 2>&1
echo "synccheck: $(grep -E 'ERROR SUMMARY' gpurun_out/san/synccheck.log | tail -1)"
