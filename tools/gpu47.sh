timeout 1800 python -m pytest tests -m gpu -q -x -k "analytic or graph_run or ess_crbd" 2>&1 | tail -3
timeout 300 python bench.py --workload crbd_vr --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
