python tools/fused_repro.py crbd 1000000
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -3
bash tools/gpu75.sh 2>&1 | tail -8
