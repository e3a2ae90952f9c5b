"""Share of ncu stall samples and instructions per code region of a capture
(diagnostic only): python tools/ncu_phase_split.py report.ncu-rep"""
import csv, io, subprocess, sys, collections
rep=sys.argv[1]
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
rows=[];f=None;hdr=None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0]=="File Path": f=r[1].split("/")[-1]; continue
    if r[0]=="Line No": hdr=r; continue
    if hdr and len(r)>6 and r[2]=="-":
        try: rows.append((f,int(r[0]),int(r[4]),int(r[7])))
        except ValueError: pass
def cat(f,l):
    if f=="lineage_warp.cuh":
        if l<=102: return "setup/batch"
        if 103<=l<=123: return "phase1 kernel"
        if 124<=l<=221: return "rounds"
        if 222<=l<=245: return "phase3"
        return "epilogue"
    if f=="lineage.cuh":
        if 95<=l<=135 or 160<=l<=225: return "phase1 main_part"
        if 136<=l<=150 or 227<=l<=250: return "node"
        return "lineage other"
    if f=="models.cuh": return "phase1 model"
    if f=="device_rng.cuh":
        if l<=40: return "philox/hq (both)"
        return "phase1 samplers"
    return f
agg=collections.defaultdict(lambda:[0,0])
for f,l,s,i in rows:
    k=cat(f,l); agg[k][0]+=s; agg[k][1]+=i
ts=sum(v[0] for v in agg.values()); ti=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(),key=lambda x:-x[1][1]): print(f"{k:22s} stall {100*v[0]/ts:5.1f}%  inst {100*v[1]/ti:5.1f}%")
