"""Per-epoch propagate / resample device time over one sweep (timing mode,
step by step), bucketed; diagnostic only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
import paper_2112_00364_b200 as smc
wl = sys.argv[1] if len(sys.argv) > 1 else "crbd"
m = {"crbd": lambda: smc.Model.crbd(inputs.tree("tree90"), lineage=True),
     "clads2": lambda: smc.Model.clads2(inputs.tree("tree90"), lineage=True),
     "seir": lambda: smc.Model.seir(inputs.seir_series()),
     "fig3": lambda: smc.Model.fig3(*inputs.FIG3_PARAMS),
     "stackf": lambda: smc.Model.stackf(inputs.stackf_series(), inputs.STACKF_PARAMS[:3] + [1024.0])}[wl]()
h = smc.Smc(m, 1_000_000, 1)
h.set_graph(False)
h.set_timing(True)
for rep in range(2):
    h.reset(1 + rep)
    prev = h.stats()
    rows = []
    while True:
        rc, done = h.step()
        st = h.stats()
        rows.append((st["ms_propagate"] - prev["ms_propagate"], st["ms_resample"] - prev["ms_resample"],
                     (st["draws"] - prev["draws"]) / 1e6))
        prev = st
        if rc or done:
            break
print(wl, "epochs", len(rows), "prop total %.2f ms" % sum(r[0] for r in rows), "resample total %.2f ms" % sum(r[1] for r in rows))
for lo, hi in ((0, 10), (10, 30), (30, 60), (60, 100), (100, 140), (140, 200)):
    sub = rows[lo:hi]
    if not sub:
        continue
    print(f"epochs {lo:3d}-{hi:3d}: prop {sum(r[0] for r in sub):7.2f} ms (mean {1e3*sum(r[0] for r in sub)/len(sub):7.1f} us)"
          f"  resample mean {1e3*sum(r[1] for r in sub)/len(sub):6.1f} us  draws/p mean {sum(r[2] for r in sub)/len(sub):6.1f}")
