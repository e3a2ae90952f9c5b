for n in 100000 300000 1000000; do python tools/fused_repro.py crbd $n; done
python tools/fused_repro.py ssm_peaked 200000
timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python tools/fused_repro.py crbd 1000000 2>&1 | head -40
timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python tools/fused_repro.py ssm_peaked 200000 2>&1 | head -30
