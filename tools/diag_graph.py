"""Sweep time: graph mode vs host-stepped (no timing) vs timing mode; wall
clock around synchronised calls, diagnostic only."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
import paper_2112_00364_b200 as smc
wl = sys.argv[1] if len(sys.argv) > 1 else "crbd"
m = {"crbd": lambda: smc.Model.crbd(inputs.tree("tree90"), lineage=True),
     "geometric": lambda: smc.Model.geometric(*inputs.GEOMETRIC_PARAMS),
     "seir": lambda: smc.Model.seir(inputs.seir_series())}[wl]()
h = smc.Smc(m, 1_000_000, 1)
def sweep(mode, seed):
    h.set_graph(mode == "graph")
    h.set_timing(mode == "timing")
    h.reset(seed)
    torch.cuda.synchronize()
    t = time.perf_counter()
    if mode == "graph":
        h.run()
    else:
        while True:
            rc, done = h.step()
            if rc or done:
                break
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3
for mode in ("graph", "step", "timing", "graph"):
    ts = [sweep(mode, s) for s in (1, 2, 3, 1, 2, 3)]
    print(wl, mode, " ".join(f"{x:.2f}" for x in ts))
