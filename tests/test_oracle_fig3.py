"""Pins of the Fig. 3(a) PCFG in the oracle (R-23): the
normalising constant of the program against the sum over its paths, the
posterior of the number of b3 visits, and the universal-control-flow
behaviour the paper describes (particles at different blocks,
reaching b_stop at different epochs)."""
import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from tests import closed_forms as cf

PRM = [0.5, 0.3, 2.0, 1.2, 1.2, 0.5]        # p_loop, p3, w1, w2, w3, w4


def test_fig3_closed_form_matches_paths():
    for prm in (PRM, [0.2, 0.5, 1.0, 2.0, 1.1, 3.0], [0.0, 0.6, 0.7, 1.0, 0.5, 1.0]):
        assert cf.fig3_z(*prm) == pytest.approx(cf.fig3_z_paths(*prm), rel=1e-10)
    assert cf.fig3_z(*PRM) == pytest.approx(5.0, rel=1e-12)


@pytest.mark.parametrize("prm", [PRM, [0.2, 0.5, 1.0, 2.0, 1.1, 3.0]])
def test_fig3_unbiased(prm):
    z = cf.fig3_z(*prm)

    def one(s):
        o = oracle.Smc(oracle.FIG3, None, prm, 1000, s)
        assert o.run() == oracle.OK
        return o.log_z

    with ThreadPoolExecutor(8) as ex:
        r = np.exp(np.array(list(ex.map(one, range(1, 301)))))
    se = r.std(ddof=1) / math.sqrt(r.size)
    assert abs(r.mean() - z) < 3 * se, (r.mean(), z, se)


def test_fig3_posterior_visits():
    # the final (unresampled) weighted particles estimate P(n | weights)
    o = oracle.Smc(oracle.FIG3, None, PRM, 200_000, 7)
    assert o.run() == oracle.OK
    n = o.fields()[:, 1].astype(int)
    w = np.exp(o.lw() - o.lw().max())
    w /= w.sum()
    ref = cf.fig3_posterior_n(PRM[0], PRM[1], PRM[4], PRM[3], 6)
    est = np.array([w[n == k].sum() for k in range(7)])
    # a few percent: SMC error at N = 2e5 is far below this, a wrong weight
    # (e.g. w3 dropped: r = 0.75) moves P(0) from 0.10 to 0.25
    np.testing.assert_allclose(est, ref, atol=0.02)


def test_fig3_control_flow():
    o = oracle.Smc(oracle.FIG3, None, PRM, 2000, 3)
    pcs, epochs_done = [], 0
    while True:
        rc, done = o.step()
        assert rc == oracle.OK
        pcs.append(o.fields()[:, 0].copy())
        epochs_done += 1
        if done:
            break
    # epoch 0 ends every particle at b1 (the b0 -> b1 checkpoint)
    assert np.all(pcs[0] == 1)
    # epoch 1: some particles stop (b4), the others wait at b2 (after b3)
    assert set(np.unique(pcs[1])) == {-1, 2}
    # particles reach b_stop at different epochs, the run ends when all have
    stopped_by = [np.mean(p == -1) for p in pcs]
    assert 0 < stopped_by[1] < 1 and stopped_by[-1] == 1.0 and epochs_done > 5
