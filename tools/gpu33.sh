for c in "constw graph" "constw step" "geometric graph" "crbd-lr graph" "crbd-seq graph"; do
  set -- $c
  timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 2 python tools/sanitize_one.py $1 $2 > gpurun_out/sc.txt 2>&1; echo "$c rc=$?"; grep -m2 -E "at void|Barrier" gpurun_out/sc.txt
done
