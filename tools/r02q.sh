export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -x -q -k "lineage or LR or clads2 or CLADS2" > gpurun_out/r02q_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02q_pytest.log
bash tools/variants.sh clads2 "" "-DSMC_PHILOX_OOL=1" "-DSMC_CLADS2_MATH_OOL=1" "-DSMC_PHILOX_OOL=1 -DSMC_CLADS2_MATH_OOL=1"
bash tools/variants.sh crbd "" "-DSMC_PHILOX_OOL=1"
O=gpurun_out/r02p2; mkdir -p $O
cap() {
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$2 --launch-skip $3 --launch-count 1 \
      -o $O/$1 -f python tools/profile_run.py --workload $4 ${@:5} > $O/$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  python tools/ncu_source.py $O/$1.ncu-rep 40 > $O/$1_source.txt 2>/dev/null
  rm -f $O/$1.ncu-rep
}
cap seir_prop_e100 propagate_kernel 100 seir
cap fig3_prop_e10 propagate_kernel 10 fig3
cap stackf_prop_e3 propagate_kernel 3 stackf
for wl in fig3 stackf; do python tools/diag_epochs.py $wl > $O/epochs_$wl.txt 2>&1; done
