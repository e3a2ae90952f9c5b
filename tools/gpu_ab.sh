# A/B: ClaDS2 merged branch-walk body, Philox unrolling (diagnostic)
O=gpurun_out/r02z5; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "clads2 or CLADS2" > $O/pytest_lr.log 2>&1; echo pytest=$?; tail -2 $O/pytest_lr.log
timeout 1500 bash tools/variants.sh clads2 "" "-DSMC_CLADS2_MERGED=0" "-DSMC_PHILOX_UNROLL=5" "" 2>&1 | tee $O/variants_clads2.txt
timeout 600 bash tools/variants.sh crbd "" "-DSMC_PHILOX_UNROLL=5" 2>&1 | tee $O/variants_crbd.txt
timeout 600 bash tools/variants.sh seir "" "-DSMC_PHILOX_UNROLL=5" 2>&1 | tee $O/variants_seir.txt
