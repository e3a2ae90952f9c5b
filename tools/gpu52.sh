timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for w in crbd crbd_vr clads2 seir geometric ssm; do timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],2), '%.4g'%d['value'], d.get('phase_ms'))"; done
