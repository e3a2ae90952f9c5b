# A/B: table sin/cos of the Box-Muller angle (diagnostic); normal-drawing models' parity first
O=gpurun_out/r02z14; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "clads2 or CLADS2 or ssm or SSM" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 900 bash tools/variants.sh clads2 "" "-DSMC_FAST_TRIG=0" "" 2>&1 | tee -a $O/variants.txt
timeout 600 bash tools/variants.sh ssm "" "-DSMC_FAST_TRIG=0" 2>&1 | tee -a $O/variants.txt
