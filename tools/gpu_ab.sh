# A/B: ClaDS2 lazy Philox peek; rolled Philox in the binomial samplers; SEIR register cap (diagnostic)
O=gpurun_out/r02z7; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "seir or clads2 or CLADS2 or seq" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 1500 bash tools/variants.sh clads2 "" "-DSMC_CLADS2_LAZYPEEK=0" "" 2>&1 | tee -a $O/variants.txt
timeout 900 bash tools/variants.sh seir "" "-DSMC_PHILOX_UNROLL_SEQ=2" "-DSMC_SEIR_MINB=3" "-DSMC_PHILOX_UNROLL_SEQ=10" 2>&1 | tee -a $O/variants.txt
EXTRA="--rng sequential" timeout 600 bash tools/variants.sh crbd "" 2>&1 | tee -a $O/variants.txt
