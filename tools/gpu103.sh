timeout 1200 python -m pytest tests/test_gpu_defer.py -x -q 2>&1 | tail -8
b() { for w in crbd; do timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done; }
b defer64
SMC_LR_DEFER_ROUNDS=0 b nodefer
SMC_LR_DEFER_ROUNDS=32 b defer32
SMC_LR_DEFER_ROUNDS=128 b defer128
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_crbd_defer2.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
