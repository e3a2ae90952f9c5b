O=gpurun_out/r02z22; mkdir -p $O
timeout 900 bash tools/variants.sh clads2 "" "-DSMC_CLADS2_SPEC_Z=0" "" "-DSMC_CLADS2_SPEC_Z=0" 2>&1 | tee -a $O/variants.txt
