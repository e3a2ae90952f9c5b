"""Whole-sweep parity at the north-star size: BASELINE configs[1]-[3] at 10^6
particles, run exactly as bench.py runs them (one CUDA-graph launch per sweep,
the fused single-launch resampling step, the same model constructors), against
one complete oracle sweep on the same seed.  The paper judges correctness by the
normalising-constant estimate (Sec. 5.1); north_star asks that
CRBD and ClaDS at 10^6 particles per GPU match the oracle.

Compared: final log Z (relative 1e-9), the final log-weights (relative 1e-9,
-inf pattern exact), the last resample's ancestors (bit-exact), every state
field (pc exact, floats relative 1e-9), and the run statistics (epochs,
resamples, alive particle-steps, helper-cap overflows, uniforms drawn: equal
for the sequential streams; ClaDS2 rate-guard
kills within a factor 2 under R-18, where their attribution is schedule-
dependent).

The four oracle sweeps (about 2-4 minutes each on one core) start together on
host threads when the first test needs them (ctypes releases the GIL).
"""
import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import inputs
import oracle
from tests.test_gpu_parity import RTOL, compare

pytestmark = pytest.mark.gpu

N = 1_000_000
SEED = 1

CASES = {
    # name: (oracle kind, data, params, GPU model constructor args)
    "crbd_lineage": (oracle.CRBD_LR, "tree90", inputs.CRBD_PARAMS, ("crbd", True)),
    "crbd_sequential": (oracle.CRBD, "tree90", inputs.CRBD_PARAMS, ("crbd", False)),
    "clads2_lineage": (oracle.CLADS2_LR, "tree90", inputs.CLADS2_PARAMS, ("clads2", True)),
    "seir": (oracle.SEIR, "seir182", None, ("seir", None)),
}


def _data(name):
    return inputs.tree("tree90") if name == "tree90" else inputs.seir_series()


def _oracle_sweep(name):
    kind, data, params, _ = CASES[name]
    d = _data(data)
    o = oracle.Smc(kind, oracle.tree_blob(d) if data == "tree90" else d, params, N, SEED)
    rc = o.run()
    return rc, o


@pytest.fixture(scope="module")
def oracle_sweeps(smc):
    ex = ThreadPoolExecutor(len(CASES))
    futs = {name: ex.submit(_oracle_sweep, name) for name in CASES}
    yield futs
    ex.shutdown(wait=True)


def _gpu_model(smc, name):
    _, data, params, (model, lineage) = CASES[name]
    if model == "crbd":
        return smc.Model.crbd(_data(data), params, lineage=lineage)
    if model == "clads2":
        return smc.Model.clads2(_data(data), params, lineage=lineage)
    return smc.Model.seir(_data(data))


@pytest.mark.parametrize("name", list(CASES))
def test_whole_sweep_10e6_vs_oracle(smc, oracle_sweeps, name):
    g = smc.Smc(_gpu_model(smc, name), N, SEED)
    assert g.resample_grid() > 0            # the fused step bench.py times
    rg = g.run_status()                     # one graph launch for the whole sweep
    ro, o = oracle_sweeps[name].result()
    assert rg == ro == oracle.OK
    assert math.isfinite(o.log_z)
    assert g.log_z == pytest.approx(o.log_z, rel=RTOL)
    compare(g, o)
    sg, so = g.stats(), o.stats()
    assert sg["epochs"] == so["epochs"] and sg["resamples"] == so["resamples"]
    assert sg["alive_particle_steps"] == so["alive_particle_steps"]
    assert sg["overflow"] == so["overflow"] == 0
    if "lineage" not in name:
        # identical streams: the GPU draws exactly the oracle's uniforms
        # (bench.py uses this count as the algorithmic work).  Under R-18 the
        # count depends on the visiting order (a detection found earlier or
        # later prunes a different number of side-tree nodes): not compared.
        assert sg["draws"] == so["draws"]
    if name == "clads2_lineage":
        # under R-18 a step whose side trees both detect and break the guard
        # may be attributed either way: only the order of magnitude is fixed
        assert so["guard"] > 0 and 0.5 < sg["guard_kills"] / so["guard"] < 2.0
    g.close()
