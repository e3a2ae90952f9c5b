"""The kernels' table-driven transcendentals — log of a uniform
(and of any positive normal double), e^x, sin/cos of 2 pi t — checked on the CPU:
the committed tables are exactly what the generators produce, and the kernels'
evaluation order (emulated with exact fma in decimal) stays within the stated
bounds of 60-digit references.  Test infrastructure only; no oracle involved."""
import math
import os
import random
import sys
from decimal import Decimal as D

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
CSRC = os.path.join(ROOT, "paper_2112_00364_b200", "csrc")

import gen_expt_table as gexp  # noqa: E402
import gen_logu_table as glog  # noqa: E402
import gen_trig_table as gtrig  # noqa: E402


def _hex_entries(path):
    txt = open(path).read()
    body = txt[txt.index("{") + 1:txt.rindex("}")]
    return [float.fromhex(t) for t in body.replace("{", " ").replace("}", " ").replace(",", " ").split()]


def test_logu_table_is_generated():
    tab = glog.table()
    got = _hex_entries(os.path.join(CSRC, "logu_table.cuh"))
    assert got == [v for row in tab for v in row]


def test_expt_table_is_generated():
    assert _hex_entries(os.path.join(CSRC, "expt_table.cuh")) == gexp.T


def test_trig_table_is_generated():
    assert _hex_entries(os.path.join(CSRC, "trig_table.cuh")) == [v for row in gtrig.TAB for v in row]


def _ulps(x, ref):
    return float(abs(D(x) - ref) / D(math.ulp(float(ref))))


def test_log_u_within_bound():
    tab = glog.table()
    rnd = random.Random(11)
    us = [rnd.random() for _ in range(1500)] + [1 - rnd.random() * 2.0 ** -rnd.randint(1, 53) for _ in range(500)] \
        + [2.0 ** -54, 1 - 2.0 ** -54, 0.5, math.sqrt(0.5)]
    worst = max(_ulps(glog.log_u(u, tab), D(u).ln()) for u in us if 0 < u < 1)
    assert worst < 1.5, worst
    # any positive normal double (log_table / log_pos)
    xs = [math.ldexp(rnd.random() + 0.5, rnd.randint(-1000, 1000)) for _ in range(1000)]
    assert max(_ulps(glog.log_u(x, tab), D(x).ln()) for x in xs) < 1.5


def test_exp_t_within_bound():
    rnd = random.Random(12)
    xs = [rnd.uniform(-30, 30) for _ in range(1500)] + [rnd.uniform(-700, 700) for _ in range(500)] + [0.0, -1e-300]
    assert max(_ulps(gexp.exp_t(x), D(x).exp()) for x in xs) < 1.5


def test_sincos2pi_within_bound():
    rnd = random.Random(13)
    ts = [rnd.random() for _ in range(1500)] + [k / 1024 for k in range(1, 1024, 7)] + [2.0 ** -54, 1 - 2.0 ** -54]
    worst = 0.0
    for t in ts:
        s, c = gtrig.sincos2pi(t)
        cs, ss = gtrig.cos_sin(2 * gtrig.PI * D(t))
        worst = max(worst, float(abs(D(c) - cs)), float(abs(D(s) - ss)))
    assert worst < 2.0 ** -52, worst


@pytest.mark.parametrize("u", [2.0 ** -54, 0.25, 0.5, 0.75, 1 - 2.0 ** -54])
def test_log_u_special_points(u):
    """Exact at the table's own points where the math is exact: log(1/2) = -ln 2 to the
    ulp, and u -> 1 keeps full relative precision (no cancellation)."""
    tab = glog.table()
    assert _ulps(glog.log_u(u, tab), D(u).ln()) < 1.5
