set -x
timeout 1200 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -15
timeout 300 python bench.py --steps 3 --warmup 3 --cpu-budget 5 2>&1 | tail -1
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_crbd.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate -s 60 -c 1 -o gpurun_out/prof_prop python tools/profile_run.py --workload crbd > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:anc_gather -s 60 -c 1 -o gpurun_out/prof_anc python tools/profile_run.py --workload crbd > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"anc_gather|reduce" -s 2 -c 2 -o gpurun_out/prof_res python tools/profile_run.py --workload resample --n 67108864 > /dev/null 2>&1
ls -la gpurun_out
