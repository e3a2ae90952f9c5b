bash tools/variants.sh crbd "" "-DSMC_FUSED_U2=4" "-DSMC_FUSED_GALLOP=1" "-DSMC_FUSED_GALLOP=1 -DSMC_FUSED_U2=4"
for fl in "" "-DSMC_FUSED_GALLOP=1"; do
  SMC_NVCC_FLAGS="$fl" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1
  SMC_NVCC_FLAGS="$fl" timeout 300 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -1
  python bench.py --workload resample --n 1048576 --steps 10 --warmup 3 --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(repr('$fl'), '2^20 ms', d['ms_per_step'], 'kernel', d['kernel_ms'])"
done
