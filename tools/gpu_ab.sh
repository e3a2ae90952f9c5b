# A/B: warp-local slot map in the fused resampling step (diagnostic); resampling tests first
O=gpurun_out/r02z11; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "fused or resample or parity or fullsweep" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 900 bash tools/variants.sh crbd "" "-DSMC_FUSED_SCAN=0" "-DSMC_CRBD_SPEC_CHILD=1" "" 2>&1 | tee -a $O/variants.txt
timeout 900 bash tools/variants.sh seir "" "-DSMC_FUSED_SCAN=0" 2>&1 | tee -a $O/variants.txt
timeout 900 bash tools/variants.sh clads2 "" "-DSMC_CLADS2_SPEC_Z=0" 2>&1 | tee -a $O/variants.txt
