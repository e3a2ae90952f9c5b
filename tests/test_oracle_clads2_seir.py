"""Pins of the oracle's ClaDS2 rate dynamics and SEIR prior block (the parts the
round-1 pins left open: alpha = 1 and sigma = 0 everywhere, fixed SEIR
parameters).  Each check compares the oracle with something computed without
it (tests/closed_forms.py, scipy's distributions):

* ClaDS2, sigma = 0, alpha != 1 (R-14): the rate-level ladder of
  backward equations (``clads2_ladder_log_lik``) on tree5, where the pending-
  rate stack holds two rates of different levels.  The ladder is itself pinned
  by its alpha = 1 reduction to the CRBD closed form and by a brute-force
  forward simulation of the generative model on a cherry.
* ClaDS2, sigma > 0: the cherry's likelihood from the forward simulation.
* ClaDS2 prior block: KS tests of the INIT draws (sigma^2 ~ InvGamma(1, 0.2),
  log alpha ~ N(0, sigma), eps ~ U(0, 1), lambda0 ~ Gamma(1, 1)) over an
  importance-sampling run (ESS threshold 0: never resampled, so the particle
  states are exactly the prior draws).
* ClaDS2 rate guard (R-14b): how often it fires at BASELINE configs[2] and
  that moving its threshold by four orders of magnitude leaves log Z alone.
* SEIR prior block (R-15): KS tests of the six Beta priors; E[Z_hat] with
  priors on a tiny population against the prior integral of the exact
  forward-algorithm likelihood (randomised Sobol points over scipy's Beta
  quantiles).

Statistical checks use the unbiasedness of SMC's Z_hat: |mean(Z_hat) - Z|
within 3 standard errors (BASELINE.json's bar), with the reference's own
Monte Carlo error added in quadrature where it has one.
"""
import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
from scipy import stats

import inputs
import oracle
from tests import closed_forms as cf

TREE5 = inputs.tree("tree5")
# two tips, root age 3 (node 0 = root)
CHERRY = {"root": 0, "parent": [-1, 0, 0], "left": [1, -1, -1], "right": [2, -1, -1],
          "age": [3.0, 0.0, 0.0]}
KINDS = [pytest.param(oracle.CLADS2, id="seq"), pytest.param(oracle.CLADS2_LR, id="lineage")]


def log_zs(kind, data, params, N, seeds, ess=None):
    """Oracle log Z over seeds (ctypes releases the GIL: runs go in parallel)."""
    def one(s):
        o = oracle.Smc(kind, data, params, N, s)
        if ess is not None:
            o.set_ess(*ess)
        rc = o.run()
        assert rc == oracle.OK
        return o.log_z
    with ThreadPoolExecutor(8) as ex:
        return np.array(list(ex.map(one, seeds)))


def check_mean_z(lz, z_ref, se_ref=0.0):
    r = np.exp(np.asarray(lz))
    se = math.sqrt(r.var(ddof=1) / r.size + se_ref * se_ref)
    assert abs(r.mean() - z_ref) < 3 * se, (r.mean(), z_ref, se)
    return r.mean(), se


# ------------------------------------------------------------ the ladder itself
def test_ladder_alpha1_is_crbd():
    # alpha = 1: every level has the same rates -> the CRBD closed form
    for lam, eps, rho in [(0.3, 1 / 3, 1.0), (0.3, 1 / 3, 0.5), (0.5, 0.0, 1.0), (0.2, 0.9, 0.7)]:
        lad = cf.clads2_ladder_log_lik(TREE5, lam, 1.0, eps, rho)
        assert lad == pytest.approx(cf.crbd_log_lik(TREE5, lam, eps * lam, rho), abs=1e-8)


def test_ladder_truncation_converged():
    for a in (0.6, 0.8, 0.95):
        assert cf.clads2_ladder_log_lik(TREE5, 0.3, a, 1 / 3, K=60) == pytest.approx(
            cf.clads2_ladder_log_lik(TREE5, 0.3, a, 1 / 3, K=100), abs=1e-9)


def test_ladder_E_yule_limit():
    # eps = 0, rho = 1: nothing goes extinct or unsampled -> E = 0 at every level
    E = cf.clads2_ladder_E(5.0, 0.7, 0.8, 0.0, 1.0)
    assert np.all(np.abs(E) < 1e-12)


def test_ladder_matches_forward_simulation():
    # sigma = 0: the brute-force forward simulation of the cherry (generative
    # model, no backward equations) agrees with the ladder
    z, se = cf.clads2_cherry_forward(3.0, 0.5, 0.8, 0.0, 0.4, 0.8, 60000, seed=7)
    lad = math.exp(cf.clads2_ladder_log_lik(CHERRY, 0.5, 0.8, 0.4, 0.8))
    assert abs(z - lad) < 3 * se, (z, lad, se)


# ------------------------------------------------------- oracle vs the ladder
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("alpha,eps,rho", [(0.8, 1 / 3, 1.0), (0.6, 0.5, 0.7)])
def test_clads2_alpha_ladder(kind, alpha, eps, rho):
    # sigma = 0 fixed, lambda0 = 0.3: params (rho, lambda0, sigma, alpha, eps)
    ref = cf.clads2_ladder_log_lik(TREE5, 0.3, alpha, eps, rho)
    lz = log_zs(kind, oracle.tree_blob(TREE5), [rho, 0.3, 0.0, alpha, eps], 1000, range(1, 601))
    check_mean_z(lz, math.exp(ref))


def test_clads2_alpha_ladder_detects_wrong_level():
    # the check above has the power to see a one-level error: the ladder
    # evaluated one level off (alpha applied once more on the observed
    # lineage) moves Z far outside 3 SE of the oracle's mean
    ref = cf.clads2_ladder_log_lik(TREE5, 0.3, 0.8, 1 / 3)
    off = cf.clads2_ladder_log_lik(TREE5, 0.3 * 0.8, 0.8, 1 / 3)
    lz = log_zs(oracle.CLADS2, oracle.tree_blob(TREE5), [1.0, 0.3, 0.0, 0.8, 1 / 3], 1000, range(1, 601))
    r = np.exp(lz)
    se = r.std(ddof=1) / math.sqrt(r.size)
    assert abs(r.mean() - math.exp(ref)) < 3 * se
    assert abs(r.mean() - math.exp(off)) > 10 * se


# --------------------------------------------- oracle vs forward simulation
@pytest.mark.parametrize("kind", KINDS)
def test_clads2_sigma_cherry_forward(kind):
    # sigma = 0.5, alpha = 0.9: lognormal rate noise at every speciation
    lam0, alpha, sigma, eps, rho = 0.5, 0.9, 0.5, 0.4, 0.8
    z, se = cf.clads2_cherry_forward(3.0, lam0, alpha, sigma, eps, rho, 60000, seed=8)
    lz = log_zs(kind, oracle.tree_blob(CHERRY), [rho, lam0, sigma, alpha, eps], 1000, range(1, 301))
    check_mean_z(lz, z, se)


# ------------------------------------------------------------- prior block
def final_fields(kind, data, params, N, seed):
    o = oracle.Smc(kind, data, params, N, seed)
    o.set_ess(0, 1)                      # importance sampling: never resampled
    assert o.run() == oracle.OK
    return o.fields()


def ks_ok(x, cdf, *args):
    p = stats.kstest(x, cdf, args=args).pvalue
    assert p > 1e-3, p


def test_clads2_prior_block():
    # fields: pc, branch, sp, sigma, alpha, eps, lam, pend[6]
    f = final_fields(oracle.CLADS2, oracle.tree_blob(CHERRY), [1.0, -1.0, -1.0, -1.0, -1.0], 40000, 3)
    sigma, alpha, eps = f[:, 3], f[:, 4], f[:, 5]
    ks_ok(sigma ** 2, "invgamma", 1.0, 0.0, 0.2)          # shape 1, scale 0.2
    ks_ok(np.log(alpha) / sigma, "norm")                  # log alpha | sigma ~ N(0, sigma)
    ks_ok(eps, "uniform")
    # lambda0 ~ Gamma(1, 1): with sigma = 0 and alpha = 1 fixed the rate never
    # changes, so the final lineage rate IS lambda0
    f = final_fields(oracle.CLADS2, oracle.tree_blob(CHERRY), [1.0, -1.0, 0.0, 1.0, -1.0], 40000, 4)
    ks_ok(f[:, 6], "gamma", 1.0, 0.0, 1.0)
    ks_ok(f[:, 5], "uniform")


SEIR_PRIORS = [(1.0, 1.0), (1 + 2 / 4.4, 3 - 2 / 4.4), (1 + 2 / 4.5, 3 - 2 / 4.5),
               (1.0, 1.0), (1 + 2 / 6.5, 3 - 2 / 6.5), (1.0, 1.0)]


def test_seir_prior_block():
    # fields 2..7: lam_h, del_h, gam_h, lam_m, del_m, rho (R-15)
    y = np.array([1.0, 0.0])
    f = final_fields(oracle.SEIR, y, [-1.0] * 6 + [3, 1, 1, 1], 40000, 6)
    for j, (a, b) in enumerate(SEIR_PRIORS):
        ks_ok(f[:, 2 + j], "beta", a, b)
    # the wrong shape order (a <-> b) for delta_h is rejected decisively
    assert stats.kstest(f[:, 3], "beta", args=SEIR_PRIORS[1][::-1]).pvalue < 1e-10


def test_seir_priors_tiny_exact():
    # E over the priors of the exact likelihood: randomised QMC (4 scrambles of
    # 2^11 Sobol points through scipy's Beta quantiles) of seir_exact_z_batch
    from scipy.stats import qmc
    y, nh, sm0, eh0, im0 = [1, 0, 1], 3, 1, 1, 1
    est = []
    for rep in range(4):
        u = qmc.Sobol(6, scramble=True, seed=100 + rep).random(2 ** 11)
        th = [stats.beta.ppf(u[:, i], a, b) for i, (a, b) in enumerate(SEIR_PRIORS)]
        est.append(float(cf.seir_exact_z_batch(y, th, nh, sm0, eh0, im0).mean()))
    z, se_q = float(np.mean(est)), float(np.std(est, ddof=1) / 2)
    lz = log_zs(oracle.SEIR, np.array(y, float), [-1.0] * 6 + [nh, sm0, eh0, im0], 2000, range(1, 401))
    check_mean_z(lz, z, se_q)


# ------------------------------------------------------------ rate guard R-14b
def test_clads2_guard_counted_and_immaterial():
    # BASELINE configs[2] (tree90, priors): the guard fires on about 1% of the
    # particle-steps (huge sigma from the InvGamma tail); log Z does not move
    # when its threshold goes from 1e4 to 1e8 (params[5]).
    t90 = oracle.tree_blob(inputs.tree("tree90"))
    prm = inputs.CLADS2_PARAMS

    def one(args):
        mr, s = args
        o = oracle.Smc(oracle.CLADS2_LR, t90, list(prm) + [mr], 3000, s)
        assert o.run() == oracle.OK
        st = o.stats()
        return mr, o.log_z, st["guard"] / st["alive_particle_steps"]

    with ThreadPoolExecutor(8) as ex:
        res = list(ex.map(one, [(mr, s) for mr in (1e4, 1e8) for s in range(1, 25)]))
    a = np.array([(lz, fr) for mr, lz, fr in res if mr == 1e4])
    b = np.array([(lz, fr) for mr, lz, fr in res if mr == 1e8])
    assert 0.002 < a[:, 1].mean() < 0.03
    se = math.sqrt(a[:, 0].var(ddof=1) / len(a) + b[:, 0].var(ddof=1) / len(b))
    assert abs(a[:, 0].mean() - b[:, 0].mean()) < 3 * se, (a[:, 0].mean(), b[:, 0].mean(), se)
