# A/B: table-driven transcendentals inside the binomial samplers (diagnostic); SEIR parity first
O=gpurun_out/r02z17; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "seir or SEIR" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 900 bash tools/variants.sh seir "" "-DSMC_FAST_BINOM=0" "" 2>&1 | tee -a $O/variants.txt
