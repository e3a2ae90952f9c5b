set -x
nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests/test_gpu_fullsweep.py -x -q --durations=10 > gpurun_out/r02b_fullsweep.log 2>&1; echo fullsweep=$?
timeout 900 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo bench=$?
timeout 600 python -m pytest tests -m gpu -x -q -k "not fullsweep" > gpurun_out/r02b_pytest.log 2>&1; echo pytest=$?
