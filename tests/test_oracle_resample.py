"""Oracle resampler pins (reading R1, DESIGN.md §R-8/§R-9).

* ancestors vs an exact-rational brute force of the systematic position rule
  (ancestor k for position j iff C_{k-1} <= (j+u)/N < C_k),
* systematic invariants: sum of offspring = N, floor(N w) <= o <= ceil(N w),
  sorted, zero-weight never selected,
* SPEC examples,
* log Z increment vs scipy's logsumexp (the plain definition of LSE),
* error cases (NaN, all -inf).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy.special import logsumexp

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def brute_ancestors(q, z):
    """Exact rationals: a_j = min{k : (j + u)/N < C_k / W}, u = (2z+1)/2^54."""
    q = [int(v) for v in q]
    N, W = len(q), sum(q)
    u = Fraction(2 * z + 1, 2 ** 54)
    C, acc = [], 0
    for v in q:
        acc += v
        C.append(acc)
    out = []
    for j in range(N):
        pos = (j + u) / N
        out.append(next(k for k in range(N) if pos < Fraction(C[k], W)))
    return np.array(out, dtype=np.uint32)


def check_invariants(q, anc):
    q = np.asarray(q, dtype=object)
    N, W = len(q), int(sum(q))
    o = np.bincount(anc.astype(np.int64), minlength=N)
    assert o.sum() == N
    assert np.all(np.diff(anc.astype(np.int64)) >= 0)
    for k in range(N):
        lo = (N * int(q[k])) // W
        hi = -((-N * int(q[k])) // W)
        assert lo <= o[k] <= hi
        if q[k] == 0:
            assert o[k] == 0


def test_brute_force_random_small():
    rng = np.random.Generator(np.random.PCG64(99))
    for case in range(400):
        N = int(rng.integers(1, 41))
        sigma = float(rng.choice([0.0, 0.5, 2.0, 6.0]))
        lw = sigma * rng.standard_normal(N)
        lw[rng.random(N) < 0.2] = -np.inf
        if not np.isfinite(lw).any():
            lw[0] = 0.0
        q = oracle.quantize(lw)
        z = int(rng.integers(0, 2 ** 53))
        anc = oracle.systematic(q, z)
        np.testing.assert_array_equal(anc, brute_ancestors(q, z))
        check_invariants(q, anc)


def test_extreme_u():
    q = np.array([3, 0, 5, 1, 0, 7], dtype=np.uint64)
    for z in (0, 1, 2 ** 52, 2 ** 53 - 1):
        anc = oracle.systematic(q, z)
        np.testing.assert_array_equal(anc, brute_ancestors(q, z))
        check_invariants(q, anc)


def test_spec_examples():
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["systematic_examples"]
    for ex in g:
        w = np.array(ex["w"])
        q = np.array([round(v * 2 ** 62) for v in w], dtype=np.uint64)
        # u = (2z+1)/2^54 closest to the example's u (exactly u + 2^-54)
        z = int(ex["u"] * 2 ** 53)
        anc = oracle.systematic(q, z)
        assert anc.tolist() == ex["anc"], ex["cite"]


def test_uniform_weights_identity():
    for N in (1, 2, 7, 1000):
        r = oracle.resample(np.full(N, -3.25), seed=5, epoch=3)
        np.testing.assert_array_equal(r["anc"], np.arange(N))
        assert r["logz_inc"] == pytest.approx(-3.25, abs=1e-14)


def test_quantization_and_logz_vs_lse():
    rng = np.random.Generator(np.random.PCG64(3))
    for N, sigma, f in [(1000, 1.0, 0.0), (5000, 4.0, 0.25), (20000, 10.0, 0.1), (3, 0.0, 0.0)]:
        lw = sigma * rng.standard_normal(N) - 7.0
        lw[rng.random(N) < f] = -np.inf
        r = oracle.resample(lw, seed=1, epoch=0)
        m = np.max(lw)
        assert r["m"] == m
        # W / 2^62 equals sum exp(lw - m) up to rounding of each q (<= 1/2 unit each)
        s = math.fsum(np.exp(lw[np.isfinite(lw)] - m))
        assert abs(Fraction(r["W"], 2 ** 62) - Fraction(s)) <= Fraction(N, 2 ** 62) + Fraction(s) * Fraction(1, 2 ** 50)
        ref = logsumexp(lw) - math.log(N)
        assert r["logz_inc"] == pytest.approx(ref, rel=1e-13, abs=1e-13)
        # u128 -> f64 conversion used for log W is truncation: exact lower bound
        Wd = oracle.u128_to_double(r["W"])
        assert Fraction(Wd) <= r["W"] and r["W"] - Fraction(Wd) < 2 ** max(0, r["W"].bit_length() - 53)


def test_resample_uses_reserved_stream():
    lw = np.random.Generator(np.random.PCG64(8)).standard_normal(300)
    seed, t = 0xDEADBEEF12345, 41
    r = oracle.resample(lw, seed=seed, epoch=t)
    blk = oracle.philox([0, t, 0, 1], [seed & 0xFFFFFFFF, seed >> 32])
    assert r["z"] == (int(blk[0]) ^ (int(blk[1]) << 21))
    np.testing.assert_array_equal(r["anc"], oracle.systematic(oracle.quantize(lw), r["z"]))


def test_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.resample(np.array([0.0, np.nan]), 1, 0)
    assert e.value.code == oracle.ENAN
    with pytest.raises(oracle.OracleError) as e:
        oracle.resample(np.array([0.0, np.inf]), 1, 0)
    assert e.value.code == oracle.ENAN
    with pytest.raises(oracle.OracleError) as e:
        oracle.resample(np.full(4, -np.inf), 1, 0)
    assert e.value.code == oracle.EREJECTED


def test_gather():
    st = np.random.Generator(np.random.PCG64(1)).integers(0, 256, (50, 64), dtype=np.uint8)
    anc = np.sort(np.random.Generator(np.random.PCG64(2)).integers(0, 50, 50)).astype(np.uint32)
    np.testing.assert_array_equal(oracle.gather(st, anc), st[anc])
