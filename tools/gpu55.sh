for sg in 0.05 0.2 0.5 1.0 2.0; do for ip in "" "--inplace"; do
timeout 300 python bench.py --workload resample --sigma $sg $ip --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sigma', d['config']['sigma'], 'inplace', d['config']['inplace'], 'ms', round(d['ms_per_step'],3), 'D/N', round(d['distinct_ancestors']/d['config']['n_per_gpu'],3), 'kernel_ms', {k: round(v,3) for k,v in d['kernel_ms'].items()})"
done; done
