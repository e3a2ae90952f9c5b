"""Minimal driver for ncu captures: one warm-up then one measured run of a
workload through the product API (never a bench number)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import inputs
import paper_2112_00364_b200 as smc

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="crbd")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--sweeps", type=int, default=1)
ap.add_argument("--rng", default="lineage")
ap.add_argument("--inplace", action="store_true")
args = ap.parse_args()
if args.workload == "resample":
    n = args.n
    dev = torch.device("cuda")
    lw = torch.randn(n, device=dev, dtype=torch.float64)
    st = torch.randint(0, 1 << 30, (16 * n,), device=dev, dtype=torch.int32)
    out = None if args.inplace else torch.empty_like(st)
    anc = torch.empty(n, device=dev, dtype=torch.int32)
    r = smc.Resampler(n, 64, 4, inplace=args.inplace)
    for e in range(1 + args.sweeps):
        r.device(lw, st, out, anc, epoch=e)
    torch.cuda.synchronize()
else:
    lin = args.rng == "lineage"
    m = {"crbd": lambda: smc.Model.crbd(inputs.tree("tree90"), lineage=lin),
         "crbd_vr": lambda: smc.Model.crbd(inputs.tree("tree90"), analytic=True),
         "clads2": lambda: smc.Model.clads2(inputs.tree("tree90"), lineage=lin),
         "seir": lambda: smc.Model.seir(inputs.seir_series()),
         "fig3": lambda: smc.Model.fig3(*inputs.FIG3_PARAMS),
         "stackf": lambda: smc.Model.stackf(inputs.stackf_series(), inputs.STACKF_PARAMS[:3] + [1024.0])}[args.workload]()
    h = smc.Smc(m, args.n, 1)
    h.set_graph(False)     # ncu does not profile kernels inside conditional-graph bodies
    if args.workload == "crbd_vr":
        h.set_ess_threshold(1, 2)
    for s in range(args.sweeps):
        h.reset(1 + s)
        h.run()
    print("logZ", h.log_z, h.stats())
