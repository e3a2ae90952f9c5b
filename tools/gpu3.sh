timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python bench.py --steps 5 --warmup 3 --cpu-budget 10 2>&1 | tail -1
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1
timeout 300 python bench.py --workload clads2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1
timeout 300 python bench.py --workload seir --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1
