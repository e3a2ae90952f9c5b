timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate -s 40 -c 1 -o gpurun_out/prof_seir python tools/profile_run.py --workload seir > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr -s 60 -c 1 -o gpurun_out/prof_clads2 python tools/profile_run.py --workload clads2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_clads2_lr3.csv python tools/profile_run.py --workload clads2 --sweeps 1 > /dev/null 2>&1
ls gpurun_out
