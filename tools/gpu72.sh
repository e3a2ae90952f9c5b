set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -x -q --durations=10 2>&1 | tail -25
timeout 300 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_default.json
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_resample.json
for w in clads2 seir crbd_vr; do timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --cpu-budget 5 2>&1 | tail -1 | tee gpurun_out/bench_$w.json; done
