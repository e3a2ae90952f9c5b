mkdir -p gpurun_out/r01i
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "resampler or crbd_tree90 or ess" 2>&1 | tail -2
rep() { python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['chain_roofline']['frac'],4), round(d['roofline']['frac'],4), {k:round(v,4) for k,v in d['kernel_ms'].items()})"; }
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 | rep cta_2p26
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 | rep cta_2p28
for w in crbd ssm; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'])"
done
SMC_NVCC_FLAGS="-DSMC_ANC_WARP" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 | rep warp_2p26
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"reduce_kernel|anc_gather" --launch-skip 2 --launch-count 2 -o gpurun_out/r01i/c4b_2p26 python tools/profile_run.py --workload resample --n 67108864 > gpurun_out/r01i/ncu_c4b.log 2>&1
