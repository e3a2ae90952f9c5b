# Evidence for a round: per-epoch phase times, cold launch lists of one sweep
# (step mode, so ncu sees every kernel), and one `ncu --set full` capture per
# dominant kernel.  Diagnostic only (numbers under a profiler are not bench values).
#   bash tools/profile_captures.sh [out-dir]   (default gpurun_out/r02f)
export PATH=/usr/local/cuda/bin:$PATH
O=${1:-gpurun_out/r02f}
mkdir -p $O
for wl in crbd clads2 seir; do python tools/diag_epochs.py $wl > $O/epochs_$wl.txt 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_crbd_sweep.csv \
    python tools/profile_run.py --workload crbd > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_clads2_sweep.csv \
    python tools/profile_run.py --workload clads2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_seir_sweep.csv \
    python tools/profile_run.py --workload seir > /dev/null 2>&1
cap() {   # name kernel-regex skip workload [extra args]
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$2 --launch-skip $3 --launch-count 1 \
      -o $O/$1 -f python tools/profile_run.py --workload $4 ${@:5} > $O/$1.log 2>&1
}
cap crbd_lrw_e3 propagate_lrw_kernel 3 crbd
cap crbd_lrw_e60 propagate_lrw_kernel 60 crbd
cap clads2_lrw_e100 propagate_lrw_kernel 100 clads2
cap crbd_fused_e100 resample_fused_kernel 100 crbd
cap seir_prop_e100 "propagate_kernel" 100 seir
cap fig3_prop_e10 "propagate_kernel" 10 fig3
cap stackf_prop_e3 "propagate_kernel" 3 stackf
cap stackf_fused_e3 resample_fused_kernel 3 stackf
cap c4_anc_gather_2p26 anc_gather_kernel 1 resample --n 67108864
ls -la $O
# export (the reports themselves are too large to bring back)
for f in $O/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
  python tools/ncu_source.py $f 40 > ${b}_source.txt 2>/dev/null
  python /root/repo/tools/ncu_phase_split.py $f > ${b}_phases.txt 2>/dev/null
done
du -sh $O/*.ncu-rep | sort -h | tail -3
rm -f $O/*.ncu-rep
