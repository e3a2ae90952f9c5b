# A/B: table log for the log(lambda) weight terms (diagnostic); birth-death parity first
O=gpurun_out/r02z13; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "crbd or clads2 or CLADS2 or lineage or analytic" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 900 bash tools/variants.sh crbd "" "-DSMC_FAST_LOGPOS=0" "" 2>&1 | tee -a $O/variants.txt
timeout 900 bash tools/variants.sh clads2 "" "-DSMC_FAST_LOGPOS=0" 2>&1 | tee -a $O/variants.txt
EXTRA="--rng sequential" timeout 900 bash tools/variants.sh crbd "" "-DSMC_FAST_LOGPOS=0" 2>&1 | tee -a $O/variants.txt
