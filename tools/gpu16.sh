for mb in 2 3 4; do
  SMC_NVCC_FLAGS="-DSMC_PROP_MINB=$mb" python paper_2112_00364_b200/csrc/build.py 2>&1 | grep -A2 "propagate_kernelINS_4Seir" | tail -1
  echo "minb=$mb"
  timeout 300 python bench.py --workload seir --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-160
  timeout 300 python bench.py --rng sequential --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-160
done
python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "seir" 2>&1 | tail -2
