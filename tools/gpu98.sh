b() { for w in $2; do timeout 300 python bench.py --workload $w --steps 3 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done; }
b base "clads2 seir"
SMC_NVCC_FLAGS="-DSMC_LR_MINB_CLADS2=5 -DSMC_SEIR_MINB=4" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b c5s4 "clads2 seir"
SMC_NVCC_FLAGS="-DSMC_LR_MINB_CLADS2=6 -DSMC_SEIR_MINB=2" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b c6s2 "clads2 seir"
SMC_NVCC_FLAGS="-DSMC_LR_MINB_CLADS2=3" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b c3 "clads2"
