mkdir -p gpurun_out/r01h
timeout 600 ncu --set full --clock-control none --import-source on -k regex:propagate_kernel --launch-skip 60 --launch-count 1 -o gpurun_out/r01h/crbdvr_mid python tools/profile_run.py --workload crbd_vr > gpurun_out/r01h/ncu_vr.log 2>&1
tail -2 gpurun_out/r01h/ncu_vr.log
for w in crbd_vr seir geometric ssm; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['value'], d.get('phase_ms'))"; done
