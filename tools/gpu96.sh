timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -x -q -k "resampler or fused" 2>&1 | tail -2
rep() { python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['chain_roofline']['frac'],4), round(d['roofline']['frac'],4), d['config'].get('state_layout','')[:12], {k:round(v,4) for k,v in d['kernel_ms'].items()})"; }
for lay in aos soa; do
timeout 300 python bench.py --workload resample --state-layout $lay --steps 10 --warmup 3 2>&1 | tail -1 | rep ${lay}_2p26
timeout 300 python bench.py --workload resample --state-layout $lay --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 | rep ${lay}_2p28
timeout 300 python bench.py --workload resample --state-layout $lay --n 1048576 --steps 20 --warmup 3 2>&1 | tail -1 | rep ${lay}_2p20
timeout 300 python bench.py --workload resample --state-layout $lay --sigma 4 --steps 10 --warmup 3 2>&1 | tail -1 | rep ${lay}_2p26_s4
done
