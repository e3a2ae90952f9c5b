timeout 1200 python -m pytest tests/test_gpu_inplace.py -q -x 2>&1 | tail -15
timeout 300 python bench.py --workload resample --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-900
timeout 300 python bench.py --workload resample --inplace --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-900
for w in crbd crbd_vr seir; do timeout 400 python bench.py --workload $w --inplace --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'inplace', round(d['ms_per_step'],2), '%.4g'%d['value'], d.get('phase_ms'))"; done
