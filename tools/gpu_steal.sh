# Work sharing at the epoch tail (lineage_warp.cuh): parity subset, per-epoch times, A/B vs no sharing.
O=gpurun_out/r02y; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "lineage or lr or clads2 or virtual" > $O/pytest_lr.log 2>&1; echo pytest=$?; tail -3 $O/pytest_lr.log
timeout 300 python tools/diag_epochs.py crbd > $O/epochs_crbd.txt 2>&1; cat $O/epochs_crbd.txt
timeout 600 python tools/diag_epochs.py clads2 > $O/epochs_clads2.txt 2>&1; cat $O/epochs_clads2.txt
timeout 900 bash tools/variants.sh crbd "-DSMC_LRW_STEAL=0" "" 2>&1 | tee $O/variants_crbd.txt
timeout 1200 bash tools/variants.sh clads2 "-DSMC_LRW_STEAL=0" "" 2>&1 | tee $O/variants_clads2.txt
