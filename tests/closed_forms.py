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


def seir_exact_z_batch(y, prm, nh, sm0, eh0=0, im0=0):
    """Exact Z(theta) of the tiny-population SEIR model for a BATCH of parameter
    vectors: prm = (lam_h, del_h, gam_h, lam_m, del_m, rho), each an array of
    shape (M,).  Same forward algorithm as ``seir_exact_log_z`` (state space
    enumerated per day, binomial pmfs from their definition); the state
    enumeration does not depend on theta (the infection probabilities
    1 - exp(-i/n_h) and the mosquito birth / survival rates are constants), so
    every probability is carried as an (M,) array.  Returns Z (not log Z)."""
    lam_h, del_h, gam_h, lam_m, del_m, rho = (np.asarray(v, dtype=np.float64) for v in prm)
    M = lam_h.shape[0]
    nu_m, mu_m = 1.0 / 7.0, 6.0 / 7.0

    def bpmf(k, n, p):                      # p: scalar or (M,) array
        return math.comb(n, k) * np.power(p, k) * np.power(1.0 - p, n - k)

    def cpmf(n, p):                         # constant-p pmf vector (length n+1)
        return np.array([math.comb(n, k) * p ** k * (1 - p) ** (n - k) for k in range(n + 1)])

    hmemo, mmemo = {}, {}

    def human(sh, eh, ih, rh, im):
        key = (sh, eh, ih, rh, im)
        if key in hmemo:
            return hmemo[key]
        out = defaultdict(lambda: np.zeros(M))
        ph = 1.0 - math.exp(-im / nh)
        for tau_h in range(sh + 1):
            p1 = math.comb(sh, tau_h) * ph ** tau_h * (1 - ph) ** (sh - tau_h)
            if p1 == 0.0:
                continue
            for de_h in range(tau_h + 1):
                p2 = p1 * bpmf(de_h, tau_h, lam_h)
                for di_h in range(eh + 1):
                    p3 = p2 * bpmf(di_h, eh, del_h)
                    for dr_h in range(ih + 1):
                        k2 = (sh - de_h, eh + de_h - di_h, ih + di_h - dr_h, rh + dr_h, di_h)
                        out[k2] = out[k2] + p3 * bpmf(dr_h, ih, gam_h)
        hmemo[key] = out
        return out

    def mosquito(sm, em, im, ih):
        key = (sm, em, im, ih)
        if key in mmemo:
            return mmemo[key]
        pm = 1.0 - math.exp(-ih / nh)
        births = cpmf(sm + em + im, nu_m)
        out = defaultdict(lambda: np.zeros(M))
        for tau_m in range(sm + 1):
            q1 = math.comb(sm, tau_m) * pm ** tau_m * (1 - pm) ** (sm - tau_m)
            if q1 == 0.0:
                continue
            for de_m in range(tau_m + 1):
                q2 = q1 * bpmf(de_m, tau_m, lam_m)
                for di_m in range(em + 1):
                    w = q2 * bpmf(di_m, em, del_m)
                    ps = np.convolve(cpmf(sm - de_m, mu_m), births)
                    pe = cpmf(em + de_m - di_m, mu_m)
                    pi = cpmf(im + di_m, mu_m)
                    for a, pa in enumerate(ps):
                        for b, pb in enumerate(pe):
                            for c, pc in enumerate(pi):
                                cst = pa * pb * pc
                                if cst != 0.0:
                                    out[(a, b, c)] = out[(a, b, c)] + w * cst
        mmemo[key] = out
        return out

    dist = {(nh - 1 - eh0, eh0, 1, 0, sm0, 0, im0): np.ones(M)}
    for yt in y:
        new = defaultdict(lambda: np.zeros(M))
        for (sh, eh, ih, rh, sm, em, im), pr in dist.items():
            H = human(sh, eh, ih, rh, im)
            Mq = mosquito(sm, em, im, ih)
            for (a, b, c, d, z), ph in H.items():
                if yt > z:
                    continue
                w = pr * ph * bpmf(yt, z, rho)
                for mk, pm_ in Mq.items():
                    k2 = (a, b, c, d) + mk
                    new[k2] = new[k2] + w * pm_
        dist = new
    return sum(dist.values())


# --------------------------------------------------------------------------
# ClaDS2 (R-14) with sigma = 0: rates are deterministic given the
# number of speciation events k a lineage descends through, lambda_k =
# alpha^k lambda0, mu_k = eps lambda_k.  The backward equations of the
# birth-death process (the CRBD E/D pair of SURVEY §8(c), with the daughters'
# rates one level up) then form a ladder:
#   dE_k/dt = mu_k - (lam_k + mu_k) E_k + lam_k E_{k+1}^2,     E_k(0) = 1 - rho
#   dD_k/dt = -(lam_k + mu_k) D_k + 2 lam_k E_{k+1} D_{k+1},   D_k(0) = rho (tips)
#   internal node c at age t_c:  D_{c,k} = lam_k D_{l,k+1} D_{r,k+1}
#   root (the INIT rate is level 0; its daughters are level 1):
#   L = D_{l,1} D_{r,1}
# Truncated at level K (level K keeps rate lam_K: a CRBD lineage).
def _clads2_rates(lam0, alpha, eps, K):
    lam = lam0 * alpha ** np.arange(K + 1, dtype=np.float64)
    return lam, eps * lam


def clads2_ladder_E(t, lam0, alpha, eps, rho, K=60):
    """E_k(t), k = 0..K (probability that a level-k lineage alive at age t
    leaves no sampled descendant)."""
    from scipy.integrate import solve_ivp
    lam, mu = _clads2_rates(lam0, alpha, eps, K)

    def f(_, E):
        up = np.append(E[1:], E[-1])
        return mu - (lam + mu) * E + lam * up * up

    if t == 0.0:
        return np.full(K + 1, 1.0 - rho)
    sol = solve_ivp(f, (0.0, t), np.full(K + 1, 1.0 - rho), rtol=1e-11, atol=1e-13, method="DOP853")
    return sol.y[:, -1]


def clads2_ladder_log_lik(tree, lam0, alpha, eps, rho=1.0, K=60):
    """log L of the fixed tree under ClaDS2 with sigma = 0 (see above)."""
    from scipy.integrate import solve_ivp
    lam, mu = _clads2_rates(lam0, alpha, eps, K)
    par, left, right, age = tree["parent"], tree["left"], tree["right"], tree["age"]
    root = tree["root"]

    def branch(c, Dc):
        """Integrate (E, D) from the child's age to the parent's age; D is kept
        normalised (returned with its log scale)."""
        tc, tp = age[c], age[par[c]]
        E0 = clads2_ladder_E(tc, lam0, alpha, eps, rho, K)

        def f(_, y):
            E, D = y[:K + 1], y[K + 1:]
            Eu = np.append(E[1:], E[-1])
            Du = np.append(D[1:], D[-1])
            return np.concatenate([mu - (lam + mu) * E + lam * Eu * Eu,
                                   -(lam + mu) * D + 2.0 * lam * Eu * Du])

        sol = solve_ivp(f, (tc, tp), np.concatenate([E0, Dc]), rtol=1e-11, atol=1e-15,
                        method="DOP853")
        return sol.y[K + 1:, -1]

    def subtree(c):
        """(D_{c,k} at the child's age, normalised; log scale)."""
        if left[c] < 0:
            return np.full(K + 1, rho), 0.0
        Dl, sl = top(left[c])
        Dr, sr = top(right[c])
        Dlu, Dru = np.append(Dl[1:], Dl[-1]), np.append(Dr[1:], Dr[-1])
        D = lam * Dlu * Dru
        m = D.max()
        return D / m, sl + sr + math.log(m)

    def top(c):
        D, s = subtree(c)
        Dt = branch(c, D)
        m = Dt.max()
        return Dt / m, s + math.log(m)

    Dl, sl = top(left[root])
    Dr, sr = top(right[root])
    return math.log(Dl[1] * Dr[1]) + sl + sr


def clads2_cherry_forward(T, lam0, alpha, sigma, eps, rho, n, seed):
    """Brute-force FORWARD simulation of the generative ClaDS2 model (not the
    SMC's backward construction): a cherry (two tips, root age T) has
    likelihood L = P(a root daughter leaves exactly one sampled extant
    descendant)^2 with the two root daughters independent (rates
    alpha lam0 e^{sigma z}).  Each daughter lineage is simulated forward to
    the present: next event after Exp(lam (1 + eps)); at the present the
    lineage is sampled with probability rho; an event is a birth with
    probability 1/(1 + eps) (two daughters with rates alpha lam e^{sigma z})
    and a death otherwise.  Returns (estimate of L, its standard error) from
    two independent halves (mean(X) * mean(Y) is unbiased for p^2)."""
    g = np.random.Generator(np.random.PCG64(seed))

    def one():
        count = 0
        stack = [(T, alpha * lam0 * math.exp(sigma * g.standard_normal()))]
        while stack:
            s, lam = stack.pop()
            while True:
                d = g.exponential(1.0 / (lam * (1.0 + eps)))
                if d > s:
                    if g.random() < rho:
                        count += 1
                        if count > 1:
                            return 0
                    break
                s -= d
                if g.random() < 1.0 / (1.0 + eps):
                    za, zb = g.standard_normal(2)
                    stack.append((s, alpha * lam * math.exp(sigma * zb)))
                    lam = alpha * lam * math.exp(sigma * za)
                    continue
                break
        return 1 if count == 1 else 0

    x = np.array([one() for _ in range(n)], dtype=np.float64)
    y = np.array([one() for _ in range(n)], dtype=np.float64)
    px, py = x.mean(), y.mean()
    se = math.sqrt(py * py * x.var(ddof=1) / n + px * px * y.var(ddof=1) / n)
    return px * py, se


# --------------------------------------------------------------------------
# The PCFG of Fig. 3(a) (R-23): b1 weights w1; every visit of b2
# draws one of {self-loop (p_loop, weight w2), b3 (p3, weight w3, back to b2),
# b4 (p4 = 1 - p_loop - p3, weight w4, stop)}.  Summing over all paths:
#   Z = w1 * sum_k (w3 B3)^k * w4 B4,   B3 = p3 / (1 - p_loop w2),
#   B4 = p4 / (1 - p_loop w2)   (the self-loops of one b2 visit sum to
#   1 / (1 - p_loop w2)),  i.e.  Z = w1 w4 B4 / (1 - w3 B3)  when w3 B3 < 1.
# The posterior of n (visits of b3) is geometric: P(n) = (1 - r) r^n, r = w3 B3.
def fig3_z(p_loop, p3, w1, w2, w3, w4):
    b3 = p3 / (1.0 - p_loop * w2)
    b4 = (1.0 - p_loop - p3) / (1.0 - p_loop * w2)
    return w1 * w4 * b4 / (1.0 - w3 * b3)


def fig3_z_paths(p_loop, p3, w1, w2, w3, w4, steps=20000):
    """The same Z by propagating the prior-weighted mass of the program's paths
    through b2, one b2 decision per step (no series summed in closed form)."""
    p4 = 1.0 - p_loop - p3
    at_b2, z = w1, 0.0
    for _ in range(steps):
        z += at_b2 * p4 * w4
        at_b2 = at_b2 * (p_loop * w2 + p3 * w3)
    return z


def fig3_posterior_n(p_loop, p3, w3, w2, nmax):
    r = w3 * p3 / (1.0 - p_loop * w2)
    return np.array([(1.0 - r) * r ** n for n in range(nmax + 1)])


# --------------------------------------------------------------------------
# STACKF (R-24): the recursive function of Fig. 5 made to terminate.
# f(p) at depth d: s ~ Gamma(p, 1/p); weight N(y_d; s, sigma) (d < |y|);
# recurse with p_rec iff s >= 1.  With D = cap // 48 frames a call from depth
# d needs frame d + 1 (allowed iff d + 2 <= D; otherwise the particle dies).
#   V_d = int_0^1 g_d(s) l_d(s) ds + [d + 2 <= D] V_{d+1} int_1^inf g_d(s) l_d(s) ds
#   Z = V_0,  g_d = Gamma(p_d, 1/p_d) density, p_0 = p0, p_d = p_rec (d >= 1).
def stackf_z(y, p0, prec, sigma, cap):
    from scipy import integrate, stats
    D = cap // 48

    def parts(d):
        p = p0 if d == 0 else prec
        g = stats.gamma(a=p, scale=1.0 / p)
        if d < len(y):
            f = lambda s: g.pdf(s) * stats.norm.pdf(y[d], loc=s, scale=sigma)   # noqa: E731
        else:
            f = g.pdf
        lo = integrate.quad(f, 0.0, 1.0, epsabs=0, epsrel=1e-12, limit=200)[0]
        hi = integrate.quad(f, 1.0, np.inf, epsabs=0, epsrel=1e-12, limit=200)[0]
        return lo, hi

    V = 0.0
    for d in range(D - 1, -1, -1):
        lo, hi = parts(d)
        V = lo + (hi * V if d + 2 <= D else 0.0)
    return V


def stackf_forward(y, p0, prec, sigma, cap, n, seed):
    """Brute-force forward simulation of the same program (numpy draws):
    returns (mean weight, its standard error) -- E[weight] = Z."""
    from scipy import stats
    g = np.random.Generator(np.random.PCG64(seed))
    D = cap // 48
    w = np.ones(n)
    alive = np.ones(n, dtype=bool)          # still recursing
    for d in range(D):
        p = p0 if d == 0 else prec
        s = g.gamma(p, 1.0 / p, size=n)
        if d < len(y):
            w = np.where(alive, w * stats.norm.pdf(y[d], loc=s, scale=sigma), w)
        rec = alive & (s >= 1.0)
        if d + 2 > D:
            w = np.where(rec, 0.0, w)       # the call would overflow the stack
            rec[:] = False
        alive = rec
    return w.mean(), w.std(ddof=1) / np.sqrt(n)
