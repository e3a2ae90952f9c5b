timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
for w in crbd crbd_vr ssm geometric; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb2', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i/launches_crbd_fused3.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
SMC_NVCC_FLAGS="-DSMC_FUSED_MINB=1" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1
for w in crbd crbd_vr ssm geometric; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i/launches_crbd_fused3_minb1.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
