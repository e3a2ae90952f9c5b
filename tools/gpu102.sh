timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "resampler" 2>&1 | tail -1
rep() { python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['chain_roofline']['frac'],4), {k:round(v,4) for k,v in d['kernel_ms'].items()})"; }
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 | rep u8_2p26
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 | rep u8_2p28
