# A/B: ClaDS2 CTAs per SM after the merged walk; captures of the one-thread-per-particle kernels
O=gpurun_out/r02f; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 bash tools/variants.sh clads2 "" "-DSMC_LRW_MINB_CLADS2=5" "-DSMC_LRW_MINB_CLADS2=6" "" 2>&1 | tee -a gpurun_out/r02z8_variants.txt
cap() {
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$2 --launch-skip $3 --launch-count 1 \
      -o $O/$1 -f python tools/profile_run.py --workload $4 ${@:5} > $O/$1.log 2>&1
}
cap seir_prop_e100 propagate_kernel 100 seir
cap fig3_prop_e10 propagate_kernel 10 fig3
cap stackf_prop_e3 propagate_kernel 3 stackf
for f in $O/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
  python tools/ncu_source.py $f 40 > ${b}_source.txt 2>/dev/null
done
rm -f $O/*.ncu-rep
