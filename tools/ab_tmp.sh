O=gpurun_out/r02z21; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "lineage or lr or clads2 or virtual" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 900 bash tools/variants.sh crbd "" "-DSMC_LRW_OVN_UNIFORM=0" "-DSMC_LRW_MINB_CRBD=6" "" 2>&1 | tee -a $O/variants.txt
timeout 900 bash tools/variants.sh clads2 "" "-DSMC_LRW_OVN_UNIFORM=0" 2>&1 | tee -a $O/variants.txt
