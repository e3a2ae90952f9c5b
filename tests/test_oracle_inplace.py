"""Pins for the in-place ancestor permutation (R-21).

The permutation c of the sorted ancestors a is fixed uniquely by four
properties, checked here without re-implementing it:
  (1) c and a hold the same multiset of ancestors;
  (2) every particle with offspring keeps its own slot: k in a => c_k = k;
  (3) the other slots ("holes") receive the remaining copies in non-decreasing
      order;
  (4) in-place safety: no hole is a source.
Exhaustive over every sorted ancestor vector for N <= 6, random at larger N;
plus SMC-level pins: a deterministic model is unchanged by the permutation,
and log Z stays unbiased (PAPER.md P:642 cites Murray et al. 2016's in-place
propagation, which RootPPL does not use).
"""
import itertools
import math

import numpy as np
import pytest

import inputs
import oracle
from tests import closed_forms as cf
from tests.test_oracle_smc import mean_ratio_within_3se, TREE5


def check_permutation(a, c):
    a = np.asarray(a)
    c = np.asarray(c)
    N = a.size
    assert sorted(c.tolist()) == sorted(a.tolist())                      # (1)
    present = np.zeros(N, bool)
    present[a] = True
    idx = np.arange(N)
    assert np.all(c[present] == idx[present])                            # (2)
    holes = ~present
    assert np.all(np.diff(c[holes].astype(np.int64)) >= 0)               # (3)
    assert not np.any(holes[c])                                          # (4)


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6])
def test_permutation_exhaustive(N):
    for a in itertools.combinations_with_replacement(range(N), N):
        check_permutation(a, oracle.permute(np.array(a, dtype=np.uint32)))


def test_permutation_random_and_special():
    rng = np.random.default_rng(5)
    for N in (7, 100, 4097):
        for sigma in (0.0, 0.5, 3.0, 20.0):
            lw = sigma * rng.standard_normal(N)
            a = oracle.resample(lw, 3, int(N + 10 * sigma))["anc"]
            check_permutation(a, oracle.permute(a))
    # identity and single survivor
    np.testing.assert_array_equal(oracle.permute(np.arange(9, dtype=np.uint32)), np.arange(9))
    c = oracle.permute(np.full(5, 3, dtype=np.uint32))
    np.testing.assert_array_equal(c, [3, 3, 3, 3, 3])
    # o = (0, 3, 2, 0, 0): 1 and 2 keep their slots, holes 0, 3, 4 get 1, 1, 2
    np.testing.assert_array_equal(oracle.permute(np.array([1, 1, 1, 2, 2], np.uint32)), [1, 1, 2, 1, 2])
    np.testing.assert_array_equal(oracle.permute(np.array([0, 0, 2, 2, 2], np.uint32)), [0, 0, 2, 2, 2])


def test_inplace_first_resample_is_permuted_plain():
    # the weights at the first checkpoint do not depend on the permutation
    a = oracle.Smc(oracle.CRBD, oracle.tree_blob(TREE5), inputs.CRBD_PARAMS, 700, 3)
    b = oracle.Smc(oracle.CRBD, oracle.tree_blob(TREE5), inputs.CRBD_PARAMS, 700, 3)
    b.set_inplace(True)
    a.step()                  # INIT (a jump) + first branch: the first checkpoint
    b.step()
    np.testing.assert_array_equal(b.anc(), oracle.permute(a.anc()))


def test_inplace_constant_weight_exact():
    s = oracle.Smc(oracle.CONSTW, None, [math.log(3.0), 4], 1000, 7)
    s.set_inplace(True)
    assert s.run() == oracle.OK
    assert s.log_z == pytest.approx(4 * math.log(3.0), abs=1e-12)


def test_inplace_crbd_unbiased():
    ref = cf.crbd_log_lik(TREE5, 0.3, 0.1)
    lz = []
    for seed in range(1, 101):
        s = oracle.Smc(oracle.CRBD, oracle.tree_blob(TREE5), [1.0, 0.3, 0.1], 1000, seed)
        s.set_inplace(True)
        s.run()
        lz.append(s.log_z)
    mean_ratio_within_3se(lz, ref)
