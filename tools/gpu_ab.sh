# A/B of build variants on the lineage-keyed kernels (diagnostic; not bench values of record)
O=gpurun_out/r02z3; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "lineage or lr or clads2 or virtual" > $O/pytest_lr.log 2>&1; echo pytest=$?; tail -2 $O/pytest_lr.log
timeout 900 bash tools/variants.sh crbd "" "-DSMC_LRW_BALLOTPUSH=0" "" "-DSMC_LRW_BALLOTPUSH=0" 2>&1 | tee $O/variants_crbd.txt
timeout 1200 bash tools/variants.sh clads2 "" "-DSMC_LRW_BALLOTPUSH=0" "" 2>&1 | tee $O/variants_clads2.txt
