timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02h_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02h_pytest.log
for wl in crbd clads2 fig3; do
  timeout 300 python bench.py --workload $wl --only --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r02h_bench_$wl.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/r02h_bench_$wl.json').read().strip().split('\n')[-1])
print('$wl', 'ms/sweep %.2f' % d['ms_per_step'], 'prop %.2f' % d['phase_ms']['propagate'], 'res %.2f' % d['phase_ms']['resample'], 'value %.3e' % d['value'])
"
done
bash tools/variants.sh clads2 "-DSMC_LRW_MINB_CLADS2=5" "-DSMC_LRW_MINB_CLADS2=6" "-DSMC_LRW_MINB_CLADS2=8"
