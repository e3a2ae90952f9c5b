timeout 900 python -m pytest tests/test_gpu_fused.py -x -q -k "aos" 2>&1 | tail -2
rep() { python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['chain_roofline']['frac'],4), round(d['roofline']['frac'],4), d['config'].get('state_layout','')[:12], {k:round(v,4) for k,v in d['kernel_ms'].items()})"; }
for lay in aos; do
timeout 300 python bench.py --workload resample --state-layout $lay --steps 10 --warmup 3 2>&1 | tail -1 | rep ${lay}_2p26
timeout 300 python bench.py --workload resample --state-layout $lay --n 268435456 --steps 5 --warmup 3 2>&1 | tail -1 | rep ${lay}_2p28
timeout 300 python bench.py --workload resample --state-layout $lay --sigma 4 --steps 10 --warmup 3 2>&1 | tail -1 | rep ${lay}_2p26_s4
timeout 300 python bench.py --workload resample --state-layout $lay --sigma 0 --steps 10 --warmup 3 2>&1 | tail -1 | rep ${lay}_2p26_s0
done
timeout 900 ncu --set full --clock-control none -k regex:"anc_gather" --launch-skip 2 --launch-count 1 -o gpurun_out/aos_2p26 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2112_00364_b200 as smc
n=1<<26
lw=torch.randn(n,device='cuda',dtype=torch.float64)
st=torch.randint(0,1<<30,(16*n,),device='cuda',dtype=torch.int32)
out=torch.empty_like(st); anc=torch.empty(n,device='cuda',dtype=torch.int32)
r=smc.Resampler(n,64,4,aos=True)
for e in range(4): r.device(lw,st,out,anc,epoch=e)
torch.cuda.synchronize()
" > /dev/null 2>&1
ncu -i gpurun_out/aos_2p26.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
for w in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']: print(w, v[h.index(w)], rows[1][h.index(w)])
"
