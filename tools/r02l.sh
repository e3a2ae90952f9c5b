timeout 900 python -m pytest tests -m gpu -x -q -k "crbd or CRBD or lineage" > gpurun_out/r02l_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02l_pytest.log
bash tools/variants.sh crbd "" "-DSMC_LRW_WMAX=8" "-DSMC_LRW_WMAX=4" "-DSMC_LRW_WMAX=2"
bash tools/variants.sh clads2 "" "-DSMC_LRW_WMAX=8" "-DSMC_LRW_WMAX=4"
