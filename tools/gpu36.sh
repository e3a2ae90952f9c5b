timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-200
