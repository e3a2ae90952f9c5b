export PATH=/usr/local/cuda/bin:$PATH
for spec in "clads2 100 e100" "crbd 60 e60" "crbd 3 e3"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:propagate_lrw_kernel --launch-skip $2 --launch-count 1 \
     -o gpurun_out/r02f_$1_$3 -f python tools/profile_run.py --workload $1 > gpurun_out/r02f_ncu_$1_$3.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:propagate --csv --log-file gpurun_out/r02f_launches_crbd.csv python tools/profile_run.py --workload crbd > /dev/null 2>&1
ls gpurun_out | grep r02f
