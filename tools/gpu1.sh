set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q --durations=15 2>&1 | tail -40
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --cpu-budget 5 2>&1 | tail -3
timeout 300 python bench.py --workload resample --steps 5 --warmup 3 2>&1 | tail -3
