# A/B: table-driven log of uniforms, 1/lambda in the CRBD walk (diagnostic); full GPU tests first
O=gpurun_out/r02z9; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
timeout 900 bash tools/variants.sh crbd "" "-DSMC_FAST_LOGU=0" "-DSMC_FAST_LOGU=0 -DSMC_CRBD_RECIP=0" "" 2>&1 | tee -a $O/variants.txt
timeout 900 bash tools/variants.sh clads2 "" "-DSMC_FAST_LOGU=0" 2>&1 | tee -a $O/variants.txt
EXTRA="--rng sequential" timeout 900 bash tools/variants.sh crbd "" "-DSMC_FAST_LOGU=0" 2>&1 | tee -a $O/variants.txt
timeout 600 bash tools/variants.sh crbd_vr "" "-DSMC_FAST_LOGU=0" 2>&1 | tee -a $O/variants.txt
