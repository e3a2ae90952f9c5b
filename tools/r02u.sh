timeout 1500 python -m pytest tests -m gpu -x -q -k "not fullsweep" > gpurun_out/r02u_pytest.log 2>&1; echo pytest=$?; tail -15 gpurun_out/r02u_pytest.log | grep -E "passed|failed|Error|assert" | head
for wl in crbd clads2 seir fig3; do
  for e in 0 1; do
    SMC_EAGER_GATHER=$e timeout 300 python bench.py --workload $wl --only --no-e2e --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().split('\n')[-1])
print('$wl eager=$e', 'ms/sweep %.2f' % d['ms_per_step'], 'prop %.2f' % d['phase_ms']['propagate'], 'res %.2f' % d['phase_ms']['resample'], 'logZ %.5f' % d['mean_log_z'])"
  done
done
