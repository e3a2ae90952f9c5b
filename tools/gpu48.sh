timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for w in crbd_vr seir geometric ssm; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['value'], d.get('phase_ms'))"; done
timeout 300 python bench.py --workload crbd --rng sequential --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
