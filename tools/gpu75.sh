mkdir -p gpurun_out/r01i
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --cpu-budget 2 2>&1 | tail -1 > gpurun_out/b75_fused.json
for w in crbd_vr clads2 seir ssm geometric; do
timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --cpu-budget 2 2>&1 | tail -1 > gpurun_out/b75_${w}_fused.json
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/b75_*.json')):
    try:
        d=json.load(open(f)); print(f, round(d['ms_per_step'],3), '%.4g'%d['value'], d.get('phase_ms'))
    except Exception as e: print(f, 'ERR', open(f).read()[:300])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i/launches_crbd_fused2.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resample_fused --launch-skip 100 --launch-count 1 -o gpurun_out/r01i/fused2_crbd_e100 python tools/profile_run.py --workload crbd > gpurun_out/r01i/ncu_fused2.log 2>&1
