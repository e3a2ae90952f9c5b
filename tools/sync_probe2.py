"""synccheck probe: is the failure order-dependent within one process?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs
import paper_2112_00364_b200 as smc
t5, t90 = inputs.tree("tree5"), inputs.tree("tree90")
first = {"lr": lambda: smc.Model.crbd(t90, lineage=True),
         "lrinp": lambda: smc.Model.crbd(t90, lineage=True, flags=smc.FLAG_INPLACE),
         "c2inp": lambda: smc.Model.clads2(t5, lineage=True, flags=smc.FLAG_INPLACE),
         "ssminp": lambda: smc.Model.ssm(inputs.ssm_series(10), flags=smc.FLAG_INPLACE)}[sys.argv[1]]()
h = smc.Smc(first, 700, 3)
h.set_graph(False)
print(sys.argv[1], h.run_status(), flush=True)
del h
h = smc.Smc(smc.Model.crbd(t5, lineage=True), 600, 4, shards=2)
h.set_graph(False)
print("then vs", h.run_status(), h.log_z, flush=True)
