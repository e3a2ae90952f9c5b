mkdir -p gpurun_out/r01i
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "resampler or shards or ess" 2>&1 | tail -2
rep() { python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['chain_roofline']['frac'],4), round(d['roofline']['frac'],4), {k:round(v,4) for k,v in d['kernel_ms'].items()})"; }
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 | rep 2p26
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 | rep 2p28
timeout 300 python bench.py --workload resample --sigma 0 --steps 10 --warmup 3 2>&1 | tail -1 | rep 2p26_sigma0
