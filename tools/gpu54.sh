mkdir -p gpurun_out/r01i
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01i/launches_inplace.csv python tools/profile_run.py --workload resample --n 67108864 --inplace > gpurun_out/r01i/p.log 2>&1
tail -3 gpurun_out/r01i/p.log
