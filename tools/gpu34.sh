timeout 900 python -m pytest tests -m gpu -q -x -k "set_data" 2>&1 | tail -3
timeout 300 python bench.py --steps 5 --warmup 3 --cpu-budget 10 2>&1 | tail -1
