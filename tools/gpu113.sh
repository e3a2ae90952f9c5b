b() { for w in crbd clads2; do timeout 300 python bench.py --workload $w --steps 3 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done; }
b t128
SMC_NVCC_FLAGS="-DSMC_LR_THREADS=64 -DSMC_LR_MINB=16 -DSMC_LR_MINB_CLADS2=8" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b t64
SMC_NVCC_FLAGS="-DSMC_LR_THREADS=96 -DSMC_LR_MINB=10 -DSMC_LR_MINB_CLADS2=5" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b t96
