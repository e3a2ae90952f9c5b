"""synccheck probe: which configuration of the cooperative kernel trips it."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs
import paper_2112_00364_b200 as smc
t5 = inputs.tree("tree5")
cfg = sys.argv[1]
n, shards = {"a": (300, 1), "b": (600, 2), "c": (256, 1), "d": (512, 2), "e": (700, 1)}[cfg]
h = smc.Smc(smc.Model.crbd(t5, lineage=True), n, 4, shards=shards)
h.set_graph(False)
print(cfg, n, shards, h.run_status(), h.log_z, flush=True)
