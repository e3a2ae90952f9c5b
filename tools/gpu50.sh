mkdir -p gpurun_out/r01h
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 200 --launch-count 120 --csv --log-file gpurun_out/r01h/launches_crbdvr.csv python tools/profile_run.py --workload crbd_vr > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 200 --launch-count 120 --csv --log-file gpurun_out/r01h/launches_crbd_lr.csv python tools/profile_run.py --workload crbd > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_kernel --launch-skip 60 --launch-count 1 -o gpurun_out/r01h/reduce_vr python tools/profile_run.py --workload crbd_vr > /dev/null 2>&1
timeout 300 python bench.py --workload crbd_vr --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-400
