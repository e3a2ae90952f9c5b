for cfg in "128 8" "64 16" "32 32"; do
  set -- $cfg
  SMC_NVCC_FLAGS="-DSMC_LR_THREADS=$1 -DSMC_LR_MINB=$2" python paper_2112_00364_b200/csrc/build.py 2>&1 | grep -A2 "propagate_lr_kernelINS_8Clads2LR" | tail -1
  echo "cfg threads=$1 minb=$2"
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-150
  timeout 300 python bench.py --workload clads2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-150
done
