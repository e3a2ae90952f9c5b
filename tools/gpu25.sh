timeout 900 python -m pytest tests -m gpu -q -x -k "resample_step or two_processes" 2>&1 | tail -3
