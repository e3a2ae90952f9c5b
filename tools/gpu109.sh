timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
rep() { python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['chain_roofline']['frac'],4), {k:round(v,4) for k,v in d['kernel_ms'].items()})"; }
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 | rep tab_2p26
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 | rep tab_2p28
for w in crbd ssm; do timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tab', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done
