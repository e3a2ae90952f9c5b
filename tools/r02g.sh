for k in warp cta; do
  for wl in crbd clads2; do
    SMC_LR_KERNEL=$k timeout 300 python bench.py --workload $wl --only --no-e2e --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().split('\n')[-1])
print('$k $wl', 'ms/sweep %.2f' % d['ms_per_step'], 'prop %.2f' % d['phase_ms']['propagate'], 'res %.2f' % d['phase_ms']['resample'], 'logZ %.4f' % d['mean_log_z'], 'draws/ps gpu %.2f' % d['draws_per_particle_step']['gpu'])
"
  done
done > gpurun_out/r02g_ab.txt 2>&1
cat gpurun_out/r02g_ab.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "lineage or LR or graph or fused or dist or engine" > gpurun_out/r02g_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02g_pytest.log
SMC_LR_KERNEL=warp python tools/diag_epochs.py crbd > gpurun_out/r02g_epochs_crbd.txt 2>&1
SMC_LR_KERNEL=warp python tools/diag_epochs.py clads2 > gpurun_out/r02g_epochs_clads2.txt 2>&1
