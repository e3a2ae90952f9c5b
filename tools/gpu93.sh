rep() { python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['chain_roofline']['frac'],4), round(d['roofline']['frac'],4), {k:round(v,4) for k,v in d['kernel_ms'].items()})"; }
b() {
for n in 262144 1048576 2097152; do
timeout 300 python bench.py --workload resample --n $n --steps 20 --warmup 3 2>&1 | tail -1 | rep $1_n$n
done
for w in crbd ssm seir; do timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'])"; done
}
b warp
SMC_NVCC_FLAGS="-DSMC_FUSED_CTA_STRIPE" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1
b cta
