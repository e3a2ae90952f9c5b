timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr -s 100 -c 1 -o gpurun_out/prof_lr_e100 python tools/profile_run.py --workload crbd > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:anc_gather -s 100 -c 1 -o gpurun_out/prof_anc_e100 python tools/profile_run.py --workload crbd > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_crbd_lr4.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
