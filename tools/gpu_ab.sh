# A/B of resampling launch shapes and the deferred gather for CRBD (diagnostic)
O=gpurun_out/r02z4; mkdir -p $O
timeout 900 bash tools/variants.sh crbd "" "-DSMC_FUSED_MINB=1" "-DSMC_FUSED_THREADS=1024 -DSMC_FUSED_MINB=1" "-DSMC_FUSED_THREADS=256 -DSMC_FUSED_MINB=4" "" 2>&1 | tee $O/variants_crbd.txt
for v in 0 1; do
  SMC_DEFERRED_GATHER=$v timeout 300 python bench.py --workload crbd --only --no-e2e --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().split('\n')[-1])
print('crbd deferred=$v ms/sweep %.2f prop %.2f res %.2f' % (d['ms_per_step'], d['phase_ms']['propagate'], d['phase_ms']['resample']))" | tee -a $O/deferred.txt
done
