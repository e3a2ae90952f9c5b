"""Run one sweep of a workload with the fused resampler (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs
import paper_2112_00364_b200 as smc
w, n = sys.argv[1], int(sys.argv[2])
m = {"crbd": lambda: smc.Model.crbd(inputs.tree("tree90"), lineage=True),
     "crbd_seq": lambda: smc.Model.crbd(inputs.tree("tree90"), lineage=False),
     "ssm_peaked": lambda: smc.Model(smc.SSM, inputs.ssm_series(50), [0.0, 100.0, 2.0, 1.0, 1e-4]),
     "seir": lambda: smc.Model.seir(inputs.seir_series())}[w]()
h = smc.Smc(m, n, 1)
h.set_graph(len(sys.argv) > 3)
print(w, n, "grid", h.resample_grid(), flush=True)
try:
    h.run()
    print("ok logZ", h.log_z)
except Exception as e:
    print("ERR", e)
