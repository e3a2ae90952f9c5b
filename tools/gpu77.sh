for n in 300000 1000000; do python tools/fused_repro.py crbd $n; done
python tools/fused_repro.py ssm_peaked 200000
timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python tools/fused_repro.py ssm_peaked 200000 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -5
bash tools/gpu75.sh 2>&1 | tail -8
