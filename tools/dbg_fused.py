"""Diagnostic: run CRBD (lineage) at N particles, print status and error message."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs
import paper_2112_00364_b200 as smc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
h = smc.Smc(smc.Model.crbd(inputs.tree("tree90"), lineage=True), n, 3)
h.set_graph(False)
try:
    h.run()
    print("ok", n, h.log_z)
except Exception as e:
    print("error", n, e)
