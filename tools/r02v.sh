timeout 1500 python -m pytest tests -m gpu -x -q -k "not fullsweep" > gpurun_out/r02v_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02v_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsweep.py -x -q > gpurun_out/r02v_fullsweep.log 2>&1; echo fullsweep=$?; tail -2 gpurun_out/r02v_fullsweep.log
for wl in stackf; do
  timeout 300 python bench.py --workload $wl --only --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r02v_bench_$wl.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r02v_bench_$wl.json').read().strip().split('\n')[-1]); print(d['ms_per_step'], d['phase_ms'], d.get('stack_copy'))"
done
