timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-230
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-230
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
timeout 900 ncu --set full --clock-control none -k regex:"reduce" -s 4 -c 1 -o gpurun_out/prof_c4b python tools/profile_run.py --workload resample --n 67108864 --sweeps 5 > /dev/null 2>&1
