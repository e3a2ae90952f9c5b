b() { for w in $2; do timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done; }
b base "crbd_vr ssm geometric"
SMC_NVCC_FLAGS="-DSMC_CRBDAE_MINB=6 -DSMC_LIGHT_MINB=8" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b m6_8 "crbd_vr ssm geometric"
SMC_NVCC_FLAGS="-DSMC_CRBDAE_MINB=8 -DSMC_LIGHT_MINB=6" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b m8_6 "crbd_vr ssm geometric"
SMC_NVCC_FLAGS="-DSMC_CRBDAE_MINB=3" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b m3 "crbd_vr"
