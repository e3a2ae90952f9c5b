mkdir -p gpurun_out/r01i
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
rep() { python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['chain_roofline']['frac'],4), round(d['roofline']['frac'],4), {k:round(v,4) for k,v in d['kernel_ms'].items()})"; }
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 | rep 2p26
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 | rep 2p28
timeout 300 python bench.py --workload resample --n 1048576 --steps 20 --warmup 3 2>&1 | tail -1 | rep 2p20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"reduce_kernel|anc_gather" --launch-skip 2 --launch-count 2 -o gpurun_out/r01i/c4c_2p26 python tools/profile_run.py --workload resample --n 67108864 > gpurun_out/r01i/ncu_c4c.log 2>&1
