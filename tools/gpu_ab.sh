# A/B: table-driven exp for the ClaDS2 rate factors (diagnostic)
O=gpurun_out/r02z10; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "clads2 or CLADS2" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 900 bash tools/variants.sh clads2 "" "-DSMC_FAST_EXP=0" "" 2>&1 | tee -a $O/variants.txt
