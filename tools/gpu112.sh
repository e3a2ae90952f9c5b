for n in 10000 100000 1000000 4000000; do
timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('crbd', $n, round(d['ms_per_step'],3), '%.4g'%d['value'], d['phase_ms'])"
done
for n in 100000 1000000; do
timeout 300 python bench.py --workload clads2 --n $n --steps 3 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('clads2', $n, round(d['ms_per_step'],3), '%.4g'%d['value'])"
done
