timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_crbd_lr.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_clads2_lr.csv python tools/profile_run.py --workload clads2 --sweeps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_seir.csv python tools/profile_run.py --workload seir --sweeps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr -s 60 -c 1 -o gpurun_out/prof_prop_lr python tools/profile_run.py --workload crbd > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr -s 3 -c 1 -o gpurun_out/prof_prop_lr_e3 python tools/profile_run.py --workload crbd > /dev/null 2>&1
ls -la gpurun_out
