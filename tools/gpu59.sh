timeout 1800 python -m pytest tests -m gpu -q -x -k "lineage or LR or graph" 2>&1 | tail -1
for w in crbd clads2; do timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],2), '%.4g'%d['value'], d.get('phase_ms'))"; done
