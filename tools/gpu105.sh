timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size" --durations=5 2>&1 | tail -10
