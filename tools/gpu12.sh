timeout 900 python -m pytest tests -m gpu -q -x -k "lineage or LR" 2>&1 | tail -2
python tools/diag_lr.py 2>&1 | head -10
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-300
cp paper_2112_00364_b200/libsmc.so /tmp/libsmc_b2.so
sed -i 's/__launch_bounds__(kLRThreads, 2)/__launch_bounds__(kLRThreads, 3)/' paper_2112_00364_b200/csrc/lineage.cuh
python paper_2112_00364_b200/csrc/build.py 2>&1 | grep -A2 "propagate_lr_kernelINS_6CrbdLR" | tail -2
python tools/diag_lr.py 2>&1 | head -10
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-300
