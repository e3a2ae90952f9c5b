timeout 900 python -m pytest tests -m gpu -x -q -k "clads2 or CLADS2" > gpurun_out/r02k_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02k_pytest.log
bash tools/variants.sh clads2 "" "-DSMC_CLADS2_SPEC_Z=1"
