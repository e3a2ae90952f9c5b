timeout 1800 python -m pytest tests -m gpu -q -x -k "lineage or LR or ess or graph or shards" 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
timeout 300 python bench.py --workload clads2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
python tools/diag_lr.py 2>&1 | head -10
