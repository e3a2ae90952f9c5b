timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json
timeout 900 python bench.py --workload crbd_vr > gpurun_out/bench_crbdvr.json 2>/dev/null; tail -1 gpurun_out/bench_crbdvr.json | cut -c1-300
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 | cut -c1-300
