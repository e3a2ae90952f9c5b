mkdir -p gpurun_out/r01i
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python tools/fused_repro.py ssm_peaked 20000 2>&1 | tail -2
timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python tools/fused_repro.py crbd 100000 2>&1 | tail -2
for w in crbd crbd_vr ssm geometric seir; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i/launches_crbd_fused5.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
SMC_NVCC_FLAGS="-DSMC_FUSED_NO_SCATTER" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1
for w in crbd ssm; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('noscatter', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i/launches_crbd_fused5_noscatter.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
