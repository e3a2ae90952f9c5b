mkdir -p gpurun_out/r01i
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i/launches_crbd_fused.csv python tools/profile_run.py --workload crbd --sweeps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resample_fused --launch-skip 100 --launch-count 1 -o gpurun_out/r01i/fused_crbd_e100 python tools/profile_run.py --workload crbd > gpurun_out/r01i/ncu_fused.log 2>&1
ls -la gpurun_out/r01i
