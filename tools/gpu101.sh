mkdir -p gpurun_out/r01i
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01i/bench_crbd.json
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/r01i/bench_resample_2p26.json
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01i/bench_resample_2p28.json
timeout 300 python bench.py --workload resample --n 1048576 --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/r01i/bench_resample_2p20.json
for w in clads2 seir crbd_vr ssm geometric; do
timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --cpu-budget 3 2>&1 | tail -1 > gpurun_out/r01i/bench_$w.json
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/r01i/bench_reference.json
