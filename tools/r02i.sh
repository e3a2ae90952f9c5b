timeout 1500 python -m pytest tests -m gpu -x -q -k "not fullsweep" > gpurun_out/r02i_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02i_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsweep.py -x -q > gpurun_out/r02i_fullsweep.log 2>&1; echo fullsweep=$?; tail -2 gpurun_out/r02i_fullsweep.log
for wl in fig3; do
  timeout 300 python bench.py --workload $wl --only --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r02i_bench_$wl.json 2>gpurun_out/r02i_bench_$wl.err
  tail -c 600 gpurun_out/r02i_bench_$wl.json
done
