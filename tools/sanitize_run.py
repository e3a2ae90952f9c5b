"""Small runs of every kernel for compute-sanitizer (memcheck/racecheck/synccheck/initcheck).

  python tools/sanitize_run.py [--step-only]

synccheck flags the first barrier of EVERY kernel launched inside the
conditional (WHILE) graph body — even the divergence-free constant-weight
kernel — and passes the identical kernels launched by the stepped loop, so it
is run with --step-only (tool limitation with conditional graph nodes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import inputs
import paper_2112_00364_b200 as smc
t5, t90 = inputs.tree("tree5"), inputs.tree("tree90")
runs = [
    ("crbd-seq", smc.Model.crbd(t90), 700),
    ("crbd-lr", smc.Model.crbd(t90, lineage=True), 700),
    ("clads2-lr", smc.Model.clads2(t5, lineage=True), 500),
    ("clads2-seq", smc.Model.clads2(t5), 300),
    ("seir", smc.Model.seir(inputs.seir_series()[:20]), 300),
    ("geometric", smc.Model.geometric(), 500),
    ("crbd-analytic", smc.Model.crbd(t90, analytic=True), 700),
    ("crbd-lr-inplace", smc.Model.crbd(t90, lineage=True, flags=smc.FLAG_INPLACE), 700),
    ("clads2-lr-inplace", smc.Model.clads2(t5, lineage=True, flags=smc.FLAG_INPLACE), 500),
    ("ssm-inplace", smc.Model.ssm(inputs.ssm_series(10), flags=smc.FLAG_INPLACE), 600),
    # several CTAs of the fused resampling kernel (grid barrier, ragged last block)
    ("crbd-lr-fused-20k", smc.Model.crbd(t90, lineage=True), 20000),
    # peaked likelihood: dominant weights take the CTA-wide (heavy) slot path
    ("ssm-peaked-fused", smc.Model(smc.SSM, inputs.ssm_series(10), [0.0, 100.0, 2.0, 1.0, 1e-4]), 20000),
]
modes = (False,) if "--step-only" in sys.argv else (False, True)
if "--shards-first" in sys.argv:
    h = smc.Smc(smc.Model.crbd(t5, lineage=True), 2 * 300, 4, shards=2)
    h.set_graph(True in modes)
    print("virtual shards", h.run_status(), h.log_z)
    del h
for name, m, n in runs:
    for graph in modes:
        h = smc.Smc(m, n, 3, shards=1)
        h.set_graph(graph)
        if "analytic" in name or ("ssm" in name and "peaked" not in name):
            h.set_ess_threshold(1, 2)             # ESS path (R-19): Sum q^2, identity copies
        rc = h.run_status()
        print(name, "graph" if graph else "step", rc, h.log_z)
if "--shards-first" not in sys.argv:
    h = smc.Smc(smc.Model.crbd(t5, lineage=True), 2 * 300, 4, shards=2)
    h.set_graph(True in modes)
    print("virtual shards", h.run_status(), h.log_z)
r = smc.Resampler(5000, 64, 1)
lw = inputs.resample_lw(5000, 2.0, 0.2, seed=1)
anc, out, inc = r.host(lw, smc.aos_to_soa(inputs.state_bytes(5000, 64, seed=2)))
print("resampler", inc)
ri = smc.Resampler(5000, 64, 1, inplace=True)
anc, out, inc = ri.host(lw, smc.aos_to_soa(inputs.state_bytes(5000, 64, seed=2)))
print("resampler in place", inc)
