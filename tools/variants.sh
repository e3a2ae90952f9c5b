# usage: [EXTRA="--rng sequential"] bash tools/variants.sh <workload> "<flags1>" "<flags2>" ...
# (diagnostic: build each variant of libsmc.so and time the workload; numbers are not bench values of record)
wl=$1; shift
for fl in "$@"; do
  SMC_NVCC_FLAGS="$fl" python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1 || { echo "build failed: $fl"; continue; }
  python bench.py --workload $wl $EXTRA --only --no-e2e --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().split('\n')[-1])
print('$wl $EXTRA', repr('$fl'), 'ms/sweep %.2f' % d['ms_per_step'], 'prop %.2f' % d.get('phase_ms',{}).get('propagate',0), 'res %.2f' % d.get('phase_ms',{}).get('resample',0))
"
done
python paper_2112_00364_b200/csrc/build.py > /dev/null 2>&1
