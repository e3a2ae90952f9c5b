timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "seir" 2>&1 | tail -2
b() { for w in seir; do timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done; }
b b256
SMC_NVCC_FLAGS="-DSMC_SEIR_BLOCK=128" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b b128
SMC_NVCC_FLAGS="-DSMC_SEIR_BLOCK=64" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b b64
SMC_NVCC_FLAGS="-DSMC_SEIR_BLOCK=32" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b b32
