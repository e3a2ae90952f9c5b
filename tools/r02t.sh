for fl in "" "-DSMC_DIAG_FUSED_NO_GATHER=1"; do
  SMC_NVCC_FLAGS="$fl" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1
  for n in 1000000 4000; do
  python bench.py --workload resample --n $n --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(repr('$fl'), $n, 'ms/step %.4f' % d['ms_per_step'], 'kernels', {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()}, 'us')"
  done
done
python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1
