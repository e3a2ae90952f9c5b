b() { for w in $2; do timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done; }
b s3 seir; b s3 seir
SMC_NVCC_FLAGS="-DSMC_SEIR_MINB=4" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b s4 seir; b s4 seir
