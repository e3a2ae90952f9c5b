python tools/diag_lr.py 2>&1 | head -10
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-400
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr -s 0 -c 1 -o gpurun_out/prof_lr_e0 python tools/profile_run.py --workload crbd > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr -s 60 -c 1 -o gpurun_out/prof_lr_e60 python tools/profile_run.py --workload crbd > /dev/null 2>&1
