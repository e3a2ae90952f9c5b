free -g | head -2
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "bench_size" --durations=3 2>&1 | tail -6
