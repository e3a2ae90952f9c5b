timeout 900 python -m pytest tests -m gpu -x -q -k "clads2 or CLADS2" > gpurun_out/r02w_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02w_pytest.log
bash tools/variants.sh clads2 "" "-DSMC_CLADS2_PIPE=0"
python tools/diag_epochs.py clads2 > gpurun_out/r02w_epochs_clads2.txt 2>&1; cat gpurun_out/r02w_epochs_clads2.txt
