for mb in 4 5 6; do
  SMC_NVCC_FLAGS="-DSMC_LR_MINB_CLADS2=$mb" python paper_2112_00364_b200/csrc/build.py 2>&1 | grep -A2 "propagate_lr_kernelINS_8Clads2LR" | tail -1
  echo "clads2 minb=$mb"
  timeout 300 python bench.py --workload clads2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-150
done
