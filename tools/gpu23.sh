timeout 300 python bench.py --workload resample --n 67108864 --steps 10 --warmup 3 2>&1 | tail -1
timeout 300 python bench.py --steps 5 --warmup 3 --cpu-budget 10 2>&1 | tail -1
