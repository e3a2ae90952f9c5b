import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
import paper_2112_00364_b200 as smc
for wl in ("crbd", "clads2"):
    m = (smc.Model.crbd if wl == "crbd" else smc.Model.clads2)(inputs.tree("tree90"), lineage=True)
    h = smc.Smc(m, 1_000_000, 1)
    h.set_graph(False)
    prev = h.stats()
    for e in range(10):
        t = time.perf_counter(); h.step(); dt = time.perf_counter() - t
        st = h.stats()
        print(wl, e, f"{dt*1e3:.2f} ms", "draws/p", round((st["draws"] - prev["draws"]) / 1e6, 1),
              "roots/p", round((st["side_roots"] - prev["side_roots"]) / 1e6, 2),
              "max_rounds", st["max_rounds"], "max_nodes", st["max_side_nodes"])
        prev = st
