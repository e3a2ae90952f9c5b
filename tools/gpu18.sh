timeout 300 python bench.py --workload seir --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
for mb in 3 4; do
  cp paper_2112_00364_b200/libsmc.so /tmp/k.so
  sed -i "s/static constexpr int kMinBlocks = 2;\(.*\)/static constexpr int kMinBlocks = $mb;\1/" paper_2112_00364_b200/csrc/models.cuh
  python paper_2112_00364_b200/csrc/build.py 2>&1 | grep -A2 "propagate_kernelINS_4Seir" | tail -1
  echo minb=$mb
  timeout 300 python bench.py --workload seir --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
  git checkout paper_2112_00364_b200/csrc/models.cuh 2>/dev/null
done
