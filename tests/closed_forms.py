"""Independent closed forms / exact enumerations used to PIN the oracle.

Test-only.  Nothing here calls the oracle or the CUDA path; each function is a
textbook result written from its mathematical definition:

* ``crbd_log_lik``  — constant-rate birth-death likelihood of a fixed
  ultrametric tree (Nee et al. 1994; the CRBD model of PAPER.md:1285-1289),
  with E(t) / g(t) as in SURVEY.md §8(c).  Itself pinned by numerical
  integration of the backward ODEs (``crbd_branch_ratio_ode``).
* ``kalman_log_z`` — exact marginal likelihood of the linear-Gaussian SSM,
  Eq. (2).
* ``seir_exact_log_z`` — forward algorithm over the enumerated state space of
  a tiny-population SEIR day step, exact binomial pmfs.
* ``geometric_z`` — sum of the series 0.5^n 1.5^(n-1).
"""
from __future__ import annotations

import math
from collections import defaultdict

import numpy as np


# --------------------------------------------------------------------------
# CRBD
def _E(t, lam, mu, rho):
    if abs(lam - mu) < 1e-15:
        return 1.0 - rho / (1.0 + rho * lam * t)
    r = lam - mu
    return 1.0 - rho * r / (rho * lam + (lam * (1 - rho) - mu) * math.exp(-r * t))


def _log_g(t, lam, mu, rho):
    if abs(lam - mu) < 1e-15:
        return -2.0 * math.log1p(rho * lam * t)
    r = lam - mu
    den = rho * lam + (lam * (1 - rho) - mu) * math.exp(-r * t)
    return -r * t - 2.0 * math.log(abs(den))


def crbd_log_lik(tree, lam, mu, rho=1.0):
    """log L = n log rho + (n-2) log lam + sum_{non-root c} log g(t_p)/g(t_c)."""
    par, left, age = tree["parent"], tree["left"], tree["age"]
    n = sum(1 for v in left if v < 0)
    s = n * math.log(rho) + (n - 2) * (math.log(lam) if lam > 0 else -math.inf)
    for c in range(len(age)):
        p = par[c]
        if p < 0:
            continue
        s += _log_g(age[p], lam, mu, rho) - _log_g(age[c], lam, mu, rho)
    return s


def crbd_branch_ratio_ode(tc, tp, lam, mu, rho):
    """log D(tp)/D(tc) by integrating dE/dt = mu - (lam+mu)E + lam E^2,
    d log D/dt = -(lam+mu) + 2 lam E from E(0) = 1 - rho (scipy RK45)."""
    from scipy.integrate import solve_ivp

    def f(t, y):
        E, _ = y
        return [mu - (lam + mu) * E + lam * E * E, -(lam + mu) + 2 * lam * E]

    sol = solve_ivp(f, (0.0, tp), [1.0 - rho, 0.0], t_eval=[tc, tp], rtol=1e-12, atol=1e-14,
                    method="DOP853")
    return sol.y[1][1] - sol.y[1][0], sol.y[0][1]


def crbd_prior_log_z(tree, rho=1.0, nodes=200):
    """log of int int L(lam, mu) Gamma(lam;1,1) Gamma(mu;1,0.5) by Gauss-Legendre
    on the prior-CDF scale (lam = -log(1-u), mu = -0.5 log(1-v))."""
    x, w = np.polynomial.legendre.leggauss(nodes)
    u = 0.5 * (x + 1.0)
    w = 0.5 * w
    lam = -np.log1p(-u)
    mu = -0.5 * np.log1p(-u)
    L = np.empty((nodes, nodes))
    for i in range(nodes):
        for j in range(nodes):
            L[i, j] = crbd_log_lik(tree, lam[i], mu[j], rho)
    m = L.max()
    return m + math.log(float(np.sum(w[:, None] * w[None, :] * np.exp(L - m))))


# --------------------------------------------------------------------------
# SSM, Eq. (2):  x0 ~ N(m0, s0^2), x_t ~ N(x_{t-1} + drift, q^2), y_t ~ N(x_t, r^2)
def kalman_log_z(y, m0=0.0, s0=100.0, drift=2.0, q=1.0, r=5.0):
    m, P = m0, s0 * s0
    ll = 0.0
    for yt in y:
        m, P = m + drift, P + q * q          # predict
        S = P + r * r
        ll += -0.5 * math.log(2 * math.pi * S) - 0.5 * (yt - m) ** 2 / S
        K = P / S                            # update
        m, P = m + K * (yt - m), (1 - K) * P
    return ll


# --------------------------------------------------------------------------
# weighted geometric (Fig. 2): Z = sum_n (1-p) p^(n-1) w^(n-1) = (1-p)/(1-p w)
def geometric_z(p, w):
    return (1 - p) / (1 - p * w)


# --------------------------------------------------------------------------
# SEIR exact forward algorithm (tiny populations)
def _binom_pmf(k, n, p):
    return math.comb(n, k) * p ** k * (1 - p) ** (n - k)


def _binom_outcomes(n, p):
    return [(k, _binom_pmf(k, n, p)) for k in range(n + 1)]


def seir_exact_log_z(y, prm, nh, sm0, eh0=0, im0=0):
    """prm = (lam_h, del_h, gam_h, lam_m, del_m, rho).  Initial state
    (sh, eh, ih, rh, sm, em, im) = (nh-1-eh0, eh0, 1, 0, sm0, 0, im0).

    Given the start-of-day state, the human and mosquito transitions use
    disjoint binomial draws, so each day factorises into a human kernel over
    (sh, eh, ih, rh, new cases) and a mosquito kernel over (sm, em, im); the
    mosquito kernel is an outer product of the three survival pmfs with the
    births pmf convolved into the susceptible axis."""
    lam_h, del_h, gam_h, lam_m, del_m, rho = prm
    nu_m, mu_m = 1.0 / 7.0, 6.0 / 7.0

    def pmf(n, p):
        return np.array([_binom_pmf(k, n, p) for k in range(n + 1)])

    def human(sh, eh, ih, rh, im):
        out = defaultdict(float)
        ph = 1.0 - math.exp(-im / nh)
        for tau_h, p1 in _binom_outcomes(sh, ph):
            for de_h, p2 in _binom_outcomes(tau_h, lam_h):
                for di_h, p3 in _binom_outcomes(eh, del_h):
                    for dr_h, p4 in _binom_outcomes(ih, gam_h):
                        key = (sh - de_h, eh + de_h - di_h, ih + di_h - dr_h, rh + dr_h, di_h)
                        out[key] += p1 * p2 * p3 * p4
        return out

    memo = {}

    def mosquito(sm, em, im, ih):
        key = (sm, em, im, ih)
        if key in memo:
            return memo[key]
        pm = 1.0 - math.exp(-ih / nh)
        nm = sm + em + im
        births = pmf(nm, nu_m)
        out = defaultdict(float)
        for tau_m, q1 in _binom_outcomes(sm, pm):
            for de_m, q2 in _binom_outcomes(tau_m, lam_m):
                for di_m, q3 in _binom_outcomes(em, del_m):
                    w = q1 * q2 * q3
                    if w == 0.0:
                        continue
                    ps = np.convolve(pmf(sm - de_m, mu_m), births)
                    pe = pmf(em + de_m - di_m, mu_m)
                    pi = pmf(im + di_m, mu_m)
                    J = w * ps[:, None, None] * pe[None, :, None] * pi[None, None, :]
                    for idx in zip(*np.nonzero(J)):
                        out[tuple(int(v) for v in idx)] += float(J[idx])
        memo[key] = out
        return out

    dist = {(nh - 1 - eh0, eh0, 1, 0, sm0, 0, im0): 1.0}
    for yt in y:
        new = defaultdict(float)
        for (sh, eh, ih, rh, sm, em, im), pr in dist.items():
            H = human(sh, eh, ih, rh, im)
            Mq = mosquito(sm, em, im, ih)
            for (a, b, c, d, z), ph in H.items():
                if yt > z:
                    continue
                w = pr * ph * _binom_pmf(yt, z, rho)
                if w == 0.0:
                    continue
                for mk, pm_ in Mq.items():
                    new[(a, b, c, d) + mk] += w * pm_
        dist = new
    return math.log(sum(dist.values()))
