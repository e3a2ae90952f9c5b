python tools/dbg_fused.py 1000; python tools/dbg_fused.py 20000; python tools/dbg_fused.py 1000000
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5 python tools/dbg_fused.py 20000 2>&1 | head -60
