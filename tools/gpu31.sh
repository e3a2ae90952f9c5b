timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 10 python tools/sanitize_run.py > gpurun_out/race.txt 2>&1; echo "race rc=$?"; tail -5 gpurun_out/race.txt
timeout 1500 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 10 python tools/sanitize_run.py > gpurun_out/sync.txt 2>&1; echo "sync rc=$?"; head -60 gpurun_out/sync.txt
