mkdir -p gpurun_out/r01i
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr --launch-skip 20 --launch-count 1 -o gpurun_out/r01i/clads2_e20 python tools/profile_run.py --workload clads2 > gpurun_out/r01i/ncu_c2.log 2>&1
tail -2 gpurun_out/r01i/ncu_c2.log
