import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs
import paper_2112_00364_b200 as smc
name, graph = sys.argv[1], sys.argv[2] == "graph"
m = {"crbd-seq": lambda: smc.Model.crbd(inputs.tree("tree90")),
     "crbd-lr": lambda: smc.Model.crbd(inputs.tree("tree90"), lineage=True),
     "geometric": lambda: smc.Model.geometric(),
     "constw": lambda: smc.Model.constw(K=3)}[name]()
h = smc.Smc(m, 700, 3)
h.set_graph(graph)
print(name, graph, h.run_status(), h.log_z)
