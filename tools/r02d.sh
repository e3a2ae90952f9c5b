bash tools/variants.sh clads2 "" "-DSMC_LR_MINB_CLADS2=6" "-DSMC_LR_MINB_CLADS2=8" > gpurun_out/r02d_variants.txt 2>&1
cat gpurun_out/r02d_variants.txt
