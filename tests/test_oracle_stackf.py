"""Pins of the STACKF program in the oracle (the compiled recursive function
of Fig. 5(c) with a byte-array PSTATE stack; R-24):
the normalising constant against the quadrature recursion and a forward
simulation of the program, the call-stack discipline (frames, return values,
stack pointer, bytes beyond the stack pointer not part of the state) and the
stack-overflow rule."""
import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import inputs
import oracle
from tests import closed_forms as cf

Y = inputs.stackf_series()
PRM = inputs.STACKF_PARAMS


def log_zs(params, N, seeds, y=Y):
    def one(s):
        o = oracle.Smc(oracle.STACKF, y, params, N, s)
        assert o.run() == oracle.OK
        return o.log_z
    with ThreadPoolExecutor(8) as ex:
        return np.array(list(ex.map(one, seeds)))


@pytest.mark.parametrize("cap", [768, 96])
def test_stackf_closed_form_vs_forward(cap):
    z = cf.stackf_z(Y, PRM[0], PRM[1], PRM[2], cap)
    m, se = cf.stackf_forward(Y, PRM[0], PRM[1], PRM[2], cap, 400_000, seed=3)
    assert abs(m - z) < 3 * se, (m, z, se)


@pytest.mark.parametrize("cap", [768, 96])
def test_stackf_unbiased(cap):
    prm = PRM[:3] + [cap]
    z = cf.stackf_z(Y, *prm)
    r = np.exp(log_zs(prm, 1000, range(1, 301)))
    se = r.std(ddof=1) / math.sqrt(r.size)
    assert abs(r.mean() - z) < 3 * se, (r.mean(), z, se)


def test_stackf_stack_discipline():
    o = oracle.Smc(oracle.STACKF, Y, PRM, 3000, 5)
    F = 48
    max_sp = 0
    while True:
        rc, done = o.step()
        assert rc == oracle.OK
        f = o.fields()
        pc, sp = f[:, 0], f[:, 1]
        live = pc != -1
        # a live particle waits at block 2 with its frames [0, sp) on the stack
        assert np.all(pc[live] == 2)
        assert np.all(sp[live] % F == 0) and np.all(sp[live] >= F)
        assert np.all(sp[~live] == 0)                       # returned to main
        frames = f[:, 3:].reshape(len(f), -1, 6)             # ra, rv, p, s1, s3, s4
        depth = (sp // F).astype(int)
        for j in range(frames.shape[1]):
            used = depth > j
            assert np.all(frames[~used, j, :] == 0.0)        # beyond sp: not state
            if used.any():
                assert np.all(frames[used, j, 0] == (-1 if j == 0 else 3))    # ra: main / block 3
                assert np.all(frames[used, j, 1] == (-1 if j == 0 else 48 * (j - 1) + 32))
                assert np.all(frames[used, j, 2] == (PRM[0] if j == 0 else PRM[1]))
        max_sp = max(max_sp, sp.max())
        if done:
            break
    # results: 64 for a leaf call, (2 r)^2 for a caller whose callee returned r
    res = o.fields()[:, 2]
    vals, r = set(), 64.0
    for _ in range(16):
        vals.add(r)
        r = (2.0 * r) ** 2 if r < 1e150 else math.inf
    fin = np.isfinite(o.lw())
    assert all(v in vals for v in res[fin])
    assert max_sp >= 3 * F


def test_stackf_overflow_rule():
    # two frames of stack: any third-level call overflows (weight -inf, counted)
    o = oracle.Smc(oracle.STACKF, Y, PRM[:3] + [96], 5000, 9)
    assert o.run() == oracle.OK
    st = o.stats()
    assert st["overflow"] > 0
    assert np.all(o.fields()[:, 1] <= 96)
