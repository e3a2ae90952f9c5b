mkdir -p gpurun_out/r01i
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
for w in crbd crbd_vr ssm geometric seir; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i/launches_crbd_fused4.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resample_fused --launch-skip 100 --launch-count 1 -o gpurun_out/r01i/fused4_crbd_e100 python tools/profile_run.py --workload crbd > gpurun_out/r01i/ncu_fused4.log 2>&1
