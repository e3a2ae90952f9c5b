mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --cpu-budget 2 2>&1 | tail -1 > gpurun_out/b73_fused.json
SMC_NO_FUSED_RESAMPLE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --cpu-budget 2 2>&1 | tail -1 > gpurun_out/b73_split.json
for w in crbd_vr clads2 seir ssm geometric; do
timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --cpu-budget 2 2>&1 | tail -1 > gpurun_out/b73_${w}_fused.json
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/b73_*.json')):
    try:
        d=json.load(open(f)); print(f, round(d['ms_per_step'],3), '%.4g'%d['value'], d.get('phase_ms'))
    except Exception as e: print(f, 'ERR', open(f).read()[:300])
PY
