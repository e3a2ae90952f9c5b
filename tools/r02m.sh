timeout 900 python -m pytest tests -m gpu -x -q -k "lineage or LR" > gpurun_out/r02m_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02m_pytest.log
bash tools/variants.sh crbd "" "-DSMC_LRW_SMEM_SLOTS=0" "-DSMC_LRW_SMEM_SLOTS=4" "-DSMC_LRW_SMEM_SLOTS=12"
bash tools/variants.sh clads2 "" "-DSMC_LRW_SMEM_SLOTS=0"
