for mb in 4 5 6 8; do
SMC_NVCC_FLAGS="-DSMC_LR_MINB_CLADS2=$mb" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1
timeout 400 python bench.py --workload clads2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb $mb', round(d['ms_per_step'],2), '%.4g'%d['value'], d.get('phase_ms'))"
done
