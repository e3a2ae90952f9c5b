"""Oracle SMC pins: the whole Alg. 1 loop (RootPPL order P:619-638)
against closed forms and exact enumeration.

SMC's normalising-constant estimate is unbiased: E[Z_hat] = Z.  Each check runs
R independent seeds and requires |mean(Z_hat/Z) - 1| < 3 SE (BASELINE.json's
statistical bar), except where the estimator is exact (constant weight).
"""
import json
import math
import os

import numpy as np
import pytest

import inputs
import oracle
from tests import closed_forms as cf

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TREE5 = inputs.tree("tree5")


def run(kind, data, params, N, seed):
    s = oracle.Smc(kind, data, params, N, seed)
    rc = s.run()
    return s, rc


def mean_ratio_within_3se(logzs, log_true):
    r = np.exp(np.asarray(logzs) - log_true)
    se = r.std(ddof=1) / math.sqrt(r.size)
    assert abs(r.mean() - 1.0) < 3 * se + 1e-12, (r.mean(), se)
    return r.mean(), se


# ---------------------------------------------------------------- closed forms
def test_crbd_closed_form_matches_ode():
    for lam, mu, rho in [(0.3, 0.1, 1.0), (0.2, 0.5, 1.0), (0.4, 0.4, 1.0), (0.4, 0.45, 1.0), (0.7, 0.0, 1.0),
                         (1.1, 0.6, 0.5)]:
        for tc, tp in [(0.0, 3.0), (2.0, 6.0), (1.5, 10.0)]:
            ode, _ = cf.crbd_branch_ratio_ode(tc, tp, lam, mu, rho)
            closed = cf._log_g(tp, lam, mu, rho) - cf._log_g(tc, lam, mu, rho)
            assert closed == pytest.approx(ode, abs=1e-9)


def test_crbd_closed_form_values():
    g = json.load(open(os.path.join(GOLD, "crbd_values.json")))
    assert cf.crbd_log_lik(TREE5, 0.3, 0.1) == pytest.approx(g["logL_fixed_lambda0.3_mu0.1"], abs=1e-12)
    # Yule special case: (n-2) log lam - lam * total branch length (= 31)
    assert cf.crbd_log_lik(TREE5, 0.5, 0.0) == pytest.approx(3 * math.log(0.5) - 0.5 * 31, abs=1e-12)
    assert cf.crbd_log_lik(TREE5, 0.5, 0.0) == pytest.approx(g["logL_yule_lambda0.5"], abs=1e-12)
    lz = cf.crbd_prior_log_z(TREE5, nodes=200)
    assert lz == pytest.approx(g["logZ_priors_gamma11_gamma1_0.5"], abs=1e-8)
    assert lz == pytest.approx(cf.crbd_prior_log_z(TREE5, nodes=400), abs=1e-10)


def test_kalman_one_step():
    # T = 1, unit variances, zero drift and mean, y = 0: y ~ N(0, 3)
    assert cf.kalman_log_z([0.0], 0.0, 1.0, 0.0, 1.0, 1.0) == pytest.approx(-0.5 * math.log(2 * math.pi * 3))


# ---------------------------------------------------------------- exact cases
@pytest.mark.parametrize("N", [1, 3, 1000])
def test_constant_weight_exact(N):
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["constw_logZ_per_checkpoint"]
    K = 4
    s, rc = run(oracle.CONSTW, None, [math.log(3.0), K], N, 7)
    assert rc == oracle.OK
    assert s.log_z == pytest.approx(K * g["value"], abs=1e-12)
    np.testing.assert_array_equal(s.anc(), np.arange(N))
    st = s.stats()
    assert st["resamples"] == K - 1 and st["epochs"] == K


def test_determinism():
    a, _ = run(oracle.CRBD, oracle.tree_blob(TREE5), inputs.CRBD_PARAMS, 300, 42)
    b, _ = run(oracle.CRBD, oracle.tree_blob(TREE5), inputs.CRBD_PARAMS, 300, 42)
    assert a.log_z == b.log_z
    np.testing.assert_array_equal(a.lw(), b.lw())
    np.testing.assert_array_equal(a.fields(), b.fields())


def test_rejected():
    # lambda = 0: log(lambda) = -inf at every internal node -> all rejected
    s, rc = run(oracle.CRBD, oracle.tree_blob(TREE5), [1.0, 0.0, 0.1], 50, 1)
    assert rc == oracle.EREJECTED and s.log_z == -math.inf


# ---------------------------------------------------------------- statistical pins
def test_weighted_geometric_unbiased():
    z = cf.geometric_z(0.5, 1.5)
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["geometric_Z"]
    assert z == g["Z"]
    lz = [run(oracle.GEOMETRIC, None, [0.5, 1.5], 1000, s)[0].log_z for s in range(1, 101)]
    mean_ratio_within_3se(lz, math.log(z))
    lz = [run(oracle.GEOMETRIC, None, [0.3, 2.0], 1000, s)[0].log_z for s in range(1, 101)]
    mean_ratio_within_3se(lz, math.log(cf.geometric_z(0.3, 2.0)))


def test_weighted_geometric_posterior():
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["geometric_posterior"]
    s, rc = run(oracle.GEOMETRIC, None, [0.5, 1.5], 100_000, 3)
    assert rc == oracle.OK
    f = s.fields()
    assert np.all(f[:, 0] == -1)                      # all at b_stop
    n = f[:, 1].astype(int)
    for k, p in enumerate(g["P"], start=1):
        assert abs(np.mean(n == k) - p) < g["tol"]
    st = s.stats()
    assert st["epochs"] > 5                            # particles finished at different epochs


def test_ssm_vs_kalman():
    y = inputs.ssm_series(10)
    ref = cf.kalman_log_z(y, *inputs.SSM_PARAMS)
    lz = [run(oracle.SSM, y, inputs.SSM_PARAMS, 2000, s)[0].log_z for s in range(1, 51)]
    mean_ratio_within_3se(lz, ref)


CRBD_KINDS = pytest.mark.parametrize("kind", [oracle.CRBD, oracle.CRBD_LR, oracle.CRBD_AE],
                                     ids=["seq", "lineage", "analytic"])


@CRBD_KINDS
@pytest.mark.parametrize("lam,mu", [(0.3, 0.1), (0.25, 0.25), (0.2, 0.4)])
def test_crbd_fixed_rates_unbiased(kind, lam, mu):
    ref = cf.crbd_log_lik(TREE5, lam, mu)
    lz = [run(kind, oracle.tree_blob(TREE5), [1.0, lam, mu], 1000, s)[0].log_z
          for s in range(1, 101)]
    mean_ratio_within_3se(lz, ref)


@CRBD_KINDS
def test_crbd_yule_unbiased(kind):
    ref = cf.crbd_log_lik(TREE5, 0.5, 0.0)
    lz = [run(kind, oracle.tree_blob(TREE5), [1.0, 0.5, 0.0], 1000, s)[0].log_z
          for s in range(1, 101)]
    mean_ratio_within_3se(lz, ref)


@CRBD_KINDS
def test_crbd_priors_unbiased(kind):
    g = json.load(open(os.path.join(GOLD, "crbd_values.json")))
    lz = [run(kind, oracle.tree_blob(TREE5), inputs.CRBD_PARAMS, 1000, s)[0].log_z
          for s in range(1, 101)]
    mean_ratio_within_3se(lz, g["logZ_priors_gamma11_gamma1_0.5"])


@CRBD_KINDS
def test_crbd_rho_half_unbiased(kind):
    # incomplete sampling (rho = 0.5): exercises the survivor Bernoulli branch
    ref = cf.crbd_log_lik(TREE5, 0.3, 0.1, rho=0.5)
    lz = [run(kind, oracle.tree_blob(TREE5), [0.5, 0.3, 0.1], 1000, s)[0].log_z
          for s in range(1, 101)]
    mean_ratio_within_3se(lz, ref)


# ---------------------------------------------------------------- §R-20 analytic E(t)
@pytest.mark.parametrize("lam,mu,rho", [(0.3, 0.1, 1.0), (0.2, 0.5, 1.0), (0.4, 0.4, 1.0), (0.4, 0.4 + 1e-9, 1.0),
                                        (0.7, 0.0, 1.0), (1.1, 0.6, 0.5), (0.2, 0.9, 0.3), (3.0, 1.0, 1.0)])
def test_crbd_E_matches_ode(lam, mu, rho):
    # E solves dE/dt = mu - (lam+mu) E + lam E^2, E(0) = 1 - rho
    for t in (1e-9, 0.01, 0.5, 3.0, 10.0):
        _, e_ode = cf.crbd_branch_ratio_ode(0.0, t, lam, mu, rho)
        e = oracle.lib().oracle_crbd_E(t, lam, mu, rho)
        assert e == pytest.approx(e_ode, rel=1e-8, abs=1e-13), (t, e, e_ode)
    assert oracle.lib().oracle_crbd_E(0.0, lam, mu, rho) == pytest.approx(1.0 - rho, abs=1e-15)


def test_crbd_E_extremes():
    E = oracle.lib().oracle_crbd_E
    assert E(1e4, 60.0, 1.0, 1.0) == pytest.approx(1.0 / 60.0, rel=1e-12)   # -> mu/lam (supercritical)
    assert E(1e4, 1.0, 60.0, 1.0) == pytest.approx(1.0, abs=1e-12)          # -> 1 (subcritical)
    assert E(5.0, 0.7, 0.0, 1.0) == 0.0                                     # Yule, complete sampling
    assert math.isfinite(E(800.0, 2.0, 1.0, 0.5)) and math.isfinite(E(800.0, 1.0, 2.0, 0.5))


def test_crbd_analytic_equals_simulated_when_E_is_zero():
    # mu = 0, rho = 1: every hidden side tree is detected (simulation) and
    # E = 0 (analytic); both kinds consume the same draws up to the first
    # hidden event, so weights, ancestors and log Z agree exactly
    a, ra = run(oracle.CRBD, oracle.tree_blob(TREE5), [1.0, 0.4, 0.0], 500, 11)
    b, rb = run(oracle.CRBD_AE, oracle.tree_blob(TREE5), [1.0, 0.4, 0.0], 500, 11)
    assert ra == rb == oracle.OK
    assert a.log_z == b.log_z
    np.testing.assert_array_equal(a.anc(), b.anc())
    np.testing.assert_array_equal(a.lw(), b.lw())


def test_crbd_analytic_reduces_variance():
    ref = cf.crbd_log_lik(TREE5, 0.3, 0.1)
    sims = [run(oracle.CRBD, oracle.tree_blob(TREE5), [1.0, 0.3, 0.1], 300, s)[0].log_z for s in range(1, 41)]
    anas = [run(oracle.CRBD_AE, oracle.tree_blob(TREE5), [1.0, 0.3, 0.1], 300, s)[0].log_z for s in range(1, 41)]
    assert np.std(anas) < np.std(sims)
    assert abs(np.mean(anas) - ref) < 0.05


def test_crbd_epochs_and_draws():
    s, rc = run(oracle.CRBD, oracle.tree_blob(TREE5), inputs.CRBD_PARAMS, 100, 9)
    st = s.stats()
    assert rc == 0 and st["epochs"] == 8 and st["resamples"] == 7   # 2n - 2 branches
    assert st["alive_particle_steps"] == 800 and st["overflow"] == 0
    f = s.fields()
    assert np.all(f[:, 0] == -1) and np.all(f[:, 1] == 8)


@pytest.mark.parametrize("kind", [oracle.CLADS2, oracle.CLADS2_LR], ids=["seq", "lineage"])
def test_clads2_reduces_to_crbd(kind):
    # sigma = 0, alpha = 1, lambda0 = 0.3, eps = 1/3  ==  CRBD(0.3, 0.1)
    ref = cf.crbd_log_lik(TREE5, 0.3, 0.1)
    lz = [run(kind, oracle.tree_blob(TREE5), [1.0, 0.3, 0.0, 1.0, 1 / 3], 1000, s)[0].log_z
          for s in range(1, 101)]
    mean_ratio_within_3se(lz, ref)


@pytest.mark.parametrize("kind", [oracle.CLADS2, oracle.CLADS2_LR], ids=["seq", "lineage"])
def test_clads2_priors_runs(kind):
    t90 = inputs.tree("tree90")
    s, rc = run(kind, oracle.tree_blob(t90), inputs.CLADS2_PARAMS, 200, 2)
    assert rc == oracle.OK and np.isfinite(s.log_z)
    st = s.stats()
    assert st["epochs"] == 178
    f = s.fields()
    assert np.all(f[:, 2] == 0)        # pending-rate stack empty at the end


@pytest.mark.parametrize("y,nh,sm0,eh0,im0", [([1, 0, 1], 3, 1, 1, 1), ([1, 0, 0], 2, 1, 1, 1)])
def test_seir_tiny_exact(y, nh, sm0, eh0, im0):
    prm = (0.5, 0.4, 0.3, 0.6, 0.5, 0.7)
    ref = cf.seir_exact_log_z(y, prm, nh, sm0, eh0, im0)
    params = list(prm) + [nh, sm0, eh0, im0]
    lz = [run(oracle.SEIR, np.array(y, float), params, 2000, s)[0].log_z for s in range(1, 101)]
    mean_ratio_within_3se(lz, ref)


def test_seir_priors_runs():
    y = inputs.seir_series()
    s, rc = run(oracle.SEIR, y, None, 200, 5)
    assert rc == oracle.OK and np.isfinite(s.log_z)
    assert s.stats()["epochs"] == len(y)
