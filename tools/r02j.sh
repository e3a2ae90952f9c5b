timeout 900 python -m pytest tests -m gpu -x -q -k "clads2 or CLADS2 or stackf or fused or inplace" > gpurun_out/r02j_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02j_pytest.log
timeout 300 python bench.py --workload stackf --only --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r02j_bench_stackf.json 2>gpurun_out/r02j_bench_stackf.err; tail -c 1500 gpurun_out/r02j_bench_stackf.json; tail -3 gpurun_out/r02j_bench_stackf.err
bash tools/variants.sh clads2 "" "-DSMC_LRW_MINB_CLADS2=5" "-DSMC_LRW_MINB_CLADS2=6" "-DSMC_LRW_MINB_CLADS2=8"
