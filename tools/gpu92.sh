timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
rep() { python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['chain_roofline']['frac'],4), round(d['roofline']['frac'],4), d['roofline']['kernel'][:25], {k:round(v,4) for k,v in d['kernel_ms'].items()})"; }
for n in 65536 262144 1048576 2097152 4194304; do
timeout 300 python bench.py --workload resample --n $n --steps 20 --warmup 3 2>&1 | tail -1 | rep n$n
SMC_NO_FUSED_RESAMPLE=1 timeout 300 python bench.py --workload resample --n $n --steps 20 --warmup 3 2>&1 | tail -1 | rep split_n$n
done
