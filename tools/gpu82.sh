mkdir -p gpurun_out/r01i
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/r01i/b82_resample.json
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01i/b82_resample_2p28.json
python -c "
import json
for f in ['gpurun_out/r01i/b82_resample.json','gpurun_out/r01i/b82_resample_2p28.json']:
    d=json.load(open(f)); print(f, d['value'], d['chain_roofline']['frac'], d['roofline']['frac'], d['kernel_ms'])
"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"reduce_kernel|anc_gather|max_kernel" --launch-skip 3 --launch-count 3 -o gpurun_out/r01i/c4_2p26 python tools/profile_run.py --workload resample --n 67108864 > gpurun_out/r01i/ncu_c4.log 2>&1
