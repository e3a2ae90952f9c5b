timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -x -q -k "lineage or LR or tree90 or full_size or clads2 or crbd" 2>&1 | tail -2
b() { for w in crbd clads2; do timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), '%.4g'%d['value'], round(d['mean_log_z'],3))"; done; }
b c4
SMC_NVCC_FLAGS="-DSMC_LR_CACHE=0" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b c0
SMC_NVCC_FLAGS="-DSMC_LR_CACHE=8" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b c8
SMC_NVCC_FLAGS="-DSMC_LR_CACHE=2" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1; b c2
