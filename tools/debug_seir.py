import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import inputs, oracle
import paper_2112_00364_b200 as smc
y = inputs.seir_series()
for graph in (False, True):
    g = smc.Smc(smc.Model.seir(y), 700, 31)
    g.set_graph(graph)
    o = oracle.Smc(oracle.SEIR, y, None, 700, 31)
    if graph:
        rc = g.run_status(); print("graph rc", rc, g.log_z, g.stats()); continue
    for e in range(60):
        rg, dg = g.step(); ro, do = o.step()
        lg, lo = g.log_weights(), o.lw()
        bad = ~np.isclose(lg, lo, rtol=1e-9) & ~(np.isneginf(lg) & np.isneginf(lo))
        print(e, rg, ro, dg, do, 'nan', np.isnan(lg).sum(), '+inf', np.isposinf(lg).sum(), 'mismatch', bad.sum(),
              'fin g/o', np.isfinite(lg).sum(), np.isfinite(lo).sum())
        if bad.any():
            i = np.nonzero(bad)[0][:3]; print('  idx', i, lg[i], lo[i]); print('  gf', g.fields()[i]); print('  of', o.fields()[i])
        if dg or do: break
