b() { for w in crbd ssm seir; do timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done;
timeout 300 python bench.py --workload resample --n 1048576 --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 resample2p20', round(d['value']), d['kernel_ms'])"; }
b t512m2
SMC_NVCC_FLAGS="-DSMC_FUSED_THREADS=256 -DSMC_FUSED_MINB=4" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b t256m4
SMC_NVCC_FLAGS="-DSMC_FUSED_THREADS=1024 -DSMC_FUSED_MINB=1" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b t1024m1
SMC_NVCC_FLAGS="-DSMC_FUSED_THREADS=256 -DSMC_FUSED_MINB=8" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b t256m8
