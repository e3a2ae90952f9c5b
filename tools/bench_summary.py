"""Print the key fields of a bench.py JSON line (diagnostic)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().split("\n")[-1])


def show(d, pre=""):
    r = d.get("roofline", {})
    rr = d.get("resample_roofline", {})
    print(f"{pre:24s} {d.get('config', {}).get('workload')}: value {d['value']:.4g} {d['unit']}, "
          f"ms/step {d['ms_per_step']:.2f}; roofline {r.get('achieved', 0):.4g}/{r.get('peak', 0):.4g} "
          f"= {r.get('frac', 0):.3f}; resample frac {rr.get('frac')}; phase {d.get('phase_ms')}; "
          f"clk {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")
    if "draws_per_particle_step" in d:
        print(" " * 26, "draws", d["draws_per_particle_step"])


show(d, "headline")
print(" " * 26, "e2e", d.get("e2e", {}).get("value"), "cpu", d.get("cpu_baseline", {}).get("value"))
for k, v in d.get("configs", {}).items():
    show(v, k)
