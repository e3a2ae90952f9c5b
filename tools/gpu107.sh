b() { for w in $2; do timeout 300 python bench.py --workload $w --steps 3 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done; }
b r1 "clads2 crbd"
SMC_NVCC_FLAGS="-DSMC_LR_RMAX=2 -DSMC_LR_ROWNERS=128" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b r2all "clads2 crbd"
SMC_NVCC_FLAGS="-DSMC_LR_RMAX=2 -DSMC_LR_ROWNERS=32" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b r2o32 "clads2"
SMC_NVCC_FLAGS="-DSMC_LR_RMAX=3 -DSMC_LR_ROWNERS=128" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b r3all "clads2"
