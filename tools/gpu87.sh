b() { for w in crbd clads2; do timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lineage or LR or tree90 or full_size" 2>&1 | tail -2
b r4o4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_crbd_r4.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
SMC_NVCC_FLAGS="-DSMC_LR_RMAX=2" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b r2o4
SMC_NVCC_FLAGS="-DSMC_LR_RMAX=4 -DSMC_LR_ROWNERS=16" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b r4o16
SMC_NVCC_FLAGS="-DSMC_LR_RMAX=1" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b r1
