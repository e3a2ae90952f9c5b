"""Oracle sampler pins: moments within 5 SE, KS/chi-
square goodness of fit against scipy's exact distributions, fixed draw counts,
special cases that reduce to a textbook routine, log-density values
and pmf normalisation."""
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
N = 200_000


def _moments(x, mean, var):
    se_m = math.sqrt(var / x.size)
    assert abs(x.mean() - mean) < 5 * se_m, (x.mean(), mean)
    # variance SE via 4th moment approximation
    se_v = math.sqrt(max(np.var((x - mean) ** 2), 1e-300) / x.size)
    assert abs(x.var() - var) < 5 * se_v + 1e-12, (x.var(), var)


def test_exp():
    x, d = oracle.sample("exp", [2.5], 11, N)
    assert np.all(d == 1)
    _moments(x, 1 / 2.5, 1 / 2.5 ** 2)
    assert stats.kstest(x, stats.expon(scale=1 / 2.5).cdf).pvalue > 1e-4


def test_bernoulli_uniform():
    x, d = oracle.sample("bernoulli", [0.3], 12, N)
    assert np.all(d == 1)
    _moments(x, 0.3, 0.21)
    x, d = oracle.sample("bernoulli", [1.0], 12, 1000)
    assert np.all(x == 1.0) and np.all(d == 1)       # S:436 degenerate, still 1 draw
    x, d = oracle.sample("uniform", [-1.0, 3.0], 13, N)
    assert np.all(d == 1) and x.min() > -1 and x.max() < 3
    assert stats.kstest(x, stats.uniform(-1, 4).cdf).pvalue > 1e-4


def test_normal():
    x, d = oracle.sample("normal", [1.5, 2.0], 14, N)
    assert np.all(d == 2)
    _moments(x, 1.5, 4.0)
    assert stats.kstest(x, stats.norm(1.5, 2.0).cdf).pvalue > 1e-4


@pytest.mark.parametrize("k,theta", [(0.4, 2.0), (1.0, 0.5), (2.3, 1.0), (30.0, 0.1)])
def test_gamma(k, theta):
    x, d = oracle.sample("gamma", [k, theta], 15, N)
    _moments(x, k * theta, k * theta * theta)
    assert stats.kstest(x, stats.gamma(k, scale=theta).cdf).pvalue > 1e-4
    if k > 1:
        assert np.all(d % 3 == 0)                   # 3 per Marsaglia-Tsang attempt
    elif k == 1:
        assert np.all(d == 1)
    else:
        assert np.all((d - 1) % 3 == 0)             # Gamma(k+1) then 1


def test_gamma_shape_one_is_exponential():
    # special case that reduces to the textbook routine: same draws, same value
    g, _ = oracle.sample("gamma", [1.0, 0.5], 16, 1000)
    e, _ = oracle.sample("exp", [2.0], 16, 1000)
    np.testing.assert_allclose(g, e, rtol=1e-15)


@pytest.mark.parametrize("a,b", [(1.0, 1.0), (1 + 2 / 4.4, 3 - 2 / 4.4), (0.5, 2.0)])
def test_beta(a, b):
    x, _ = oracle.sample("beta", [a, b], 17, N)
    _moments(x, a / (a + b), a * b / ((a + b) ** 2 * (a + b + 1)))
    assert stats.kstest(x, stats.beta(a, b).cdf).pvalue > 1e-4


@pytest.mark.parametrize("n,p", [(0, 0.3), (7, 0.0), (7, 1.0), (20, 0.2), (40, 0.6),
                                 (1000, 0.3), (73700, 1 / 7), (73700, 6 / 7), (7369, 1e-4)])
def test_binomial_chi_square(n, p):
    M = 100_000
    x, d = oracle.sample("binomial", [n, p], 18, M)
    assert np.all(x == np.floor(x)) and x.min() >= 0 and x.max() <= n
    pp = p if p <= 0.5 else 1 - p
    if n * pp < 10:
        assert np.all(d == 1)                       # inversion: exactly 1 draw
    else:
        assert np.all(d % 2 == 0)                   # BTRS: 2 per attempt
    if n == 0 or p in (0.0, 1.0):
        assert np.all(x == (n if p == 1.0 else 0))
        return
    # chi-square on bins with expected count >= 20 (tails pooled)
    k = np.arange(n + 1)
    pmf = stats.binom.pmf(k, n, p)
    obs = np.bincount(x.astype(np.int64), minlength=n + 1).astype(float)
    exp = pmf * M
    keep = exp >= 20
    o = np.append(obs[keep], obs[~keep].sum())
    e = np.append(exp[keep], exp[~keep].sum())
    if e[-1] < 5:
        o, e = o[:-1], e[:-1]
        e *= o.sum() / e.sum()
    chi2 = ((o - e) ** 2 / e).sum()
    assert stats.chi2.sf(chi2, len(o) - 1) > 1e-4


def test_log_densities():
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["normal_logpdf"]
    assert oracle.normal_logpdf(0.0, 0.0, 1.0) == pytest.approx(g["at0"], abs=g["tol"])
    assert oracle.normal_logpdf(0.3, 0.0, 1.0) == pytest.approx(g["at03"], abs=g["tol"])
    for y, mu, s in [(1.2, -0.3, 2.5), (10.0, 3.0, 5.0)]:
        assert oracle.normal_logpdf(y, mu, s) == pytest.approx(stats.norm(mu, s).logpdf(y), rel=1e-13)


def test_binomial_logpmf():
    for n, p in [(0, 0.3), (1, 0.5), (12, 0.3), (500, 0.01), (7370, 0.3)]:
        lp = np.array([oracle.binomial_logpmf(k, n, p) for k in range(n + 1)])
        # S:450 asks 1e-12; the lgamma form loses ~eps*lgamma(n+1) absolute in log space
        tol = max(1e-12, 4 * np.finfo(float).eps * math.lgamma(n + 1))
        assert abs(math.fsum(np.exp(lp)) - 1.0) < tol
        ks = np.arange(0, n + 1, max(1, n // 50))
        ref = stats.binom.logpmf(ks, n, p)
        np.testing.assert_allclose(lp[ks][np.isfinite(ref)], ref[np.isfinite(ref)], rtol=1e-10,
                                   atol=1e-10)
    assert oracle.binomial_logpmf(3, 2, 0.5) == -math.inf
    assert oracle.binomial_logpmf(0, 5, 0.0) == 0.0
    assert oracle.binomial_logpmf(5, 5, 1.0) == 0.0
