timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr -s 100 -c 1 -o gpurun_out/prof_lr128_e100 python tools/profile_run.py --workload crbd > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr -s 3 -c 1 -o gpurun_out/prof_lr128_e3 python tools/profile_run.py --workload crbd > /dev/null 2>&1
