mkdir -p gpurun_out/r01i
timeout 300 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01i/bench_crbd.json
timeout 300 python bench.py --workload resample --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/r01i/bench_resample_2p26.json
timeout 300 python bench.py --workload resample --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01i/bench_resample_2p28.json
for w in clads2 seir crbd_vr ssm geometric; do
timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --cpu-budget 3 2>&1 | tail -1 > gpurun_out/r01i/bench_$w.json
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i/launches_crbd_sweep.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i/launches_resample_2p26.csv python tools/profile_run.py --workload resample --n 67108864 --sweeps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resample_fused --launch-skip 100 --launch-count 1 -o gpurun_out/r01i/prof_fused_e100 python tools/profile_run.py --workload crbd > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"reduce_kernel|anc_gather|max_kernel" --launch-skip 3 --launch-count 3 -o gpurun_out/r01i/prof_c4_2p26 python tools/profile_run.py --workload resample --n 67108864 > /dev/null 2>&1
ls gpurun_out/r01i
