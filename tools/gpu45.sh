python tools/diag_epochs.py crbd
python tools/diag_epochs.py clads2
python tools/diag_epochs.py seir
mkdir -p gpurun_out/r01h
timeout 900 ncu --set full --clock-control none --import-source on -k regex:propagate_lr --launch-skip 60 --launch-count 1 -o gpurun_out/r01h/crbd_mid python tools/profile_run.py --workload crbd > gpurun_out/r01h/ncu.log 2>&1
tail -3 gpurun_out/r01h/ncu.log
