mkdir -p gpurun_out/r01j
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_kernel --launch-skip 90 --launch-count 1 -o gpurun_out/r01j/seir_e90 python tools/profile_run.py --workload seir > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr --launch-skip 100 --launch-count 1 -o gpurun_out/r01j/clads2_e100 python tools/profile_run.py --workload clads2 > /dev/null 2>&1
ls gpurun_out/r01j
