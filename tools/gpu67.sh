mkdir -p gpurun_out/san
for tool in memcheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/$tool.log | tail -2)"
done
grep -E "Error|Uninit|Race" gpurun_out/san/initcheck.log gpurun_out/san/racecheck.log | sort | uniq -c | sort -rn | head -5
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py --step-only > gpurun_out/san/synccheck.log 2>&1; echo "synccheck: $(grep -E "ERROR SUMMARY" gpurun_out/san/synccheck.log | tail -1)"
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 400 python bench.py --workload clads2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],2), '%.4g'%d['value'], d.get('phase_ms'))"
