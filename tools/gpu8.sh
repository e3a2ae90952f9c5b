timeout 1500 python -m pytest tests -m gpu -q -x -k "lineage or LR or graph or shards" 2>&1 | tail -3
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1
timeout 600 python bench.py --workload clads2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_crbd_lr2.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
