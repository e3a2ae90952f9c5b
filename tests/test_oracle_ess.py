"""ESS-adaptive resampling.

Pins: the ESS examples of S:510-512; the exact integer gate against Python
big integers; unbiasedness of the normalising-constant estimate for several
thresholds (closed forms: CRBD, weighted geometric, Kalman); tau = 0 is plain
importance sampling and tau >= 1 the plain Algorithm 1."""
import json
import math
import os

import numpy as np
import pytest

import inputs
import oracle
from tests import closed_forms as cf
from tests.test_oracle_smc import mean_ratio_within_3se

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TREE5 = inputs.tree("tree5")


def test_ess_examples():
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["ess_examples"]
    for ex in g:
        _, ess = oracle.ess_gate(np.log(np.asarray(ex["w"])), 1, 1)
        assert ess == pytest.approx(ex["ess"], rel=1e-12), ex["cite"]
    lw = np.full(7, -np.inf)
    lw[3] = -2.0
    assert oracle.ess_gate(lw, 1, 1)[1] == pytest.approx(1.0)      # single finite weight


def test_gate_exact_vs_bigint():
    rng = np.random.default_rng(5)
    for case in range(300):
        N = int(rng.integers(1, 60))
        lw = float(rng.choice([0.1, 1.0, 5.0])) * rng.standard_normal(N)
        lw[rng.random(N) < 0.2] = -np.inf
        if not np.isfinite(lw).any():
            lw[0] = 0.0
        a, b = int(rng.integers(0, 12)), int(rng.integers(1, 12))
        q = [int(v) for v in oracle.quantize(lw)]
        W, Q2 = sum(q), sum(v * v for v in q)
        expect = a >= b or b * W * W < a * N * Q2
        assert oracle.ess_gate(lw, a, b)[0] == expect


def run_ess(kind, data, params, N, seed, a, b):
    s = oracle.Smc(kind, data, params, N, seed)
    s.set_ess(a, b)
    rc = s.run()
    return s, rc


@pytest.mark.parametrize("kind", [oracle.CRBD, oracle.CRBD_LR], ids=["seq", "lineage"])
@pytest.mark.parametrize("a,b", [(1, 2), (0, 1), (9, 10)])
def test_crbd_unbiased_with_ess(kind, a, b):
    ref = cf.crbd_log_lik(TREE5, 0.3, 0.1)
    runs = [run_ess(kind, oracle.tree_blob(TREE5), [1.0, 0.3, 0.1], 1000, s, a, b) for s in range(1, 101)]
    mean_ratio_within_3se([r[0].log_z for r in runs], ref)
    res = [r[0].stats()["resamples"] for r in runs]
    if a == 0:
        assert max(res) == 0                         # tau = 0: importance sampling
    else:
        assert max(res) <= 7


@pytest.mark.parametrize("a,b", [(1, 2), (0, 1)])
def test_geometric_and_ssm_unbiased_with_ess(a, b):
    lz = [run_ess(oracle.GEOMETRIC, None, [0.5, 1.5], 1000, s, a, b)[0].log_z for s in range(1, 101)]
    mean_ratio_within_3se(lz, math.log(2.0))
    y = inputs.ssm_series(10)
    ref = cf.kalman_log_z(y, *inputs.SSM_PARAMS)
    lz = [run_ess(oracle.SSM, y, inputs.SSM_PARAMS, 2000, s, a, b)[0].log_z for s in range(1, 51)]
    mean_ratio_within_3se(lz, ref)


def test_constant_weight_exact_any_tau():
    for a, b in [(0, 1), (1, 2), (1, 1), (5, 3)]:
        s, rc = run_ess(oracle.CONSTW, None, [math.log(3.0), 4], 100, 1, a, b)
        assert rc == 0 and s.log_z == pytest.approx(4 * math.log(3.0), abs=1e-12)
        # equal weights: ESS = N, so only tau >= 1 resamples
        assert s.stats()["resamples"] == (3 if a >= b else 0)


def test_tau_zero_is_importance_sampling():
    # never resample: log Z = log mean of the total weights = LSE(lw_final) - log N
    y = inputs.ssm_series(10)
    s, rc = run_ess(oracle.SSM, y, inputs.SSM_PARAMS, 500, 3, 0, 1)
    assert rc == 0 and s.stats()["resamples"] == 0
    lw = s.lw()
    f = lw[np.isfinite(lw)]
    ref = np.log(np.sum(np.exp(f - f.max()))) + f.max() - math.log(500)
    assert s.log_z == pytest.approx(ref, rel=1e-12)
