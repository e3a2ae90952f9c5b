"""BASELINE.json's statistical bar: over 100 independent runs the mean
normalising-constant estimate of the GPU matches the oracle's within 3 SE
(seeds 1-100 on the GPU, 101-200 on the oracle), and both match the CRBD
closed form on config C0 (tree5, N = 1000)."""
import json
import math
import multiprocessing
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import inputs
import oracle
from tests import closed_forms as cf

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _oracle_logz(args):
    kind, data, params, N, seed = args
    s = oracle.Smc(kind, data, params, N, seed)
    s.run()
    return s.log_z


def oracle_runs(kind, data, params, N, seeds):
    ctx = multiprocessing.get_context("spawn")          # never fork a CUDA process
    with ProcessPoolExecutor(max_workers=min(8, os.cpu_count() or 1), mp_context=ctx) as ex:
        return list(ex.map(_oracle_logz, [(kind, data, params, N, s) for s in seeds]))


def gpu_runs(smc, model, N, seeds):
    h = smc.Smc(model, N, seeds[0])
    out = []
    for s in seeds:
        h.reset(s)
        h.run()
        out.append(h.log_z)
    return out


def ratio_stats(lz, ref):
    r = np.exp(np.asarray(lz) - ref)
    return r.mean(), r.std(ddof=1) / math.sqrt(r.size)


@pytest.mark.parametrize("lineage", [False, True], ids=["seq", "lineage"])
@pytest.mark.parametrize("params,which", [(inputs.CRBD_PARAMS, "priors"), ([1.0, 0.3, 0.1], "fixed")])
def test_c0_gpu_vs_oracle_vs_closed_form(smc, lineage, params, which):
    tree = inputs.tree("tree5")
    g = json.load(open(os.path.join(GOLD, "crbd_values.json")))
    ref = (g["logZ_priors_gamma11_gamma1_0.5"] if which == "priors"
           else cf.crbd_log_lik(tree, 0.3, 0.1))
    gl = gpu_runs(smc, smc.Model.crbd(tree, params, lineage=lineage), 1000, list(range(1, 101)))
    ol = oracle_runs(oracle.CRBD_LR if lineage else oracle.CRBD, oracle.tree_blob(tree), params, 1000,
                     list(range(101, 201)))
    mg, sg = ratio_stats(gl, ref)
    mo, so = ratio_stats(ol, ref)
    assert abs(mg - 1) < 3 * sg, (mg, sg)                  # GPU vs closed form
    assert abs(mo - 1) < 3 * so, (mo, so)                  # oracle vs closed form
    assert abs(mg - mo) < 3 * math.hypot(sg, so), (mg, mo)  # GPU vs oracle


@pytest.mark.parametrize("lineage", [False, True], ids=["seq", "lineage"])
def test_tree90_gpu_vs_oracle(smc, lineage):
    """configs[1] tree, N = 10^4: mean log Z of 100 GPU runs vs 100 oracle runs
    (same N, so the same small-N bias; compared on the log scale)."""
    tree = inputs.tree("tree90")
    gl = np.array(gpu_runs(smc, smc.Model.crbd(tree, lineage=lineage), 10_000, list(range(1, 101))))
    ol = np.array(oracle_runs(oracle.CRBD_LR if lineage else oracle.CRBD, oracle.tree_blob(tree),
                              inputs.CRBD_PARAMS, 10_000, list(range(101, 201))))
    se = math.hypot(gl.std(ddof=1), ol.std(ddof=1)) / 10.0
    assert abs(gl.mean() - ol.mean()) < 3 * se, (gl.mean(), ol.mean(), se)
