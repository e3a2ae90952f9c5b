timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
cp paper_2112_00364_b200/libsmc.so /tmp/keep.so
for cfg in "64 16" "128 10"; do
  set -- $cfg
  SMC_NVCC_FLAGS="-DSMC_LR_THREADS=$1 -DSMC_LR_MINB=$2" python paper_2112_00364_b200/csrc/build.py 2>&1 | grep -A2 "propagate_lr_kernelINS_6CrbdLR" | tail -1
  echo "cfg threads=$1 minb=$2"
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-140
done
cp /tmp/keep.so paper_2112_00364_b200/libsmc.so
timeout 300 python bench.py --steps 5 --warmup 3 --cpu-budget 10 2>&1 | tail -1
