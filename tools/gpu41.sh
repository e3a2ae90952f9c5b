for w in geometric ssm seir clads2; do timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --cpu-budget 5 2>&1 | tail -1 | cut -c1-330; done
