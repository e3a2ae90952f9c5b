set -x
export PATH=/usr/local/cuda/bin:$PATH
python tools/diag_epochs.py clads2 > gpurun_out/r02c_epochs_clads2.txt 2>&1
python tools/diag_epochs.py crbd > gpurun_out/r02c_epochs_crbd.txt 2>&1
for spec in "clads2 100 e100" "clads2 4 e4" "crbd 60 e60" "crbd 3 e3"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:propagate_lr_kernel --launch-skip $2 --launch-count 1 \
     -o gpurun_out/r02c_$1_$3 -f python tools/profile_run.py --workload $1 > gpurun_out/r02c_ncu_$1_$3.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:resample_fused_kernel --launch-skip 100 --launch-count 1 \
     -o gpurun_out/r02c_fused_crbd_e100 -f python tools/profile_run.py --workload crbd > gpurun_out/r02c_ncu_fused.log 2>&1
ls -la gpurun_out
