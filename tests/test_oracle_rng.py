"""Oracle RNG pins: Philox4x32-10 known answers (Random123), the uniform
conversion's range/distribution, and the stream layout (DESIGN.md §R-1/§R-2)."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_known_answers():
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for c in kat["cases"]:
        ctr = [int(x, 16) for x in c["ctr"]]
        key = [int(x, 16) for x in c["key"]]
        out = oracle.philox(ctr, key)
        assert [int(x) for x in out] == [int(x, 16) for x in c["out"]]


def test_uniform_open_interval_and_distribution():
    from scipy import stats
    u = oracle.uniforms(seed=7, particle=3, epoch=2, tag=0, n=200_000)
    assert u.min() > 0.0 and u.max() < 1.0
    assert stats.kstest(u, "uniform").pvalue > 1e-4
    # independence of consecutive draws (both halves of a block and across blocks)
    r = np.corrcoef(u[:-1], u[1:])[0, 1]
    assert abs(r) < 5 / np.sqrt(u.size)


def test_uniform_resolution():
    # u = (2z+1) 2^-54 is exactly representable whenever z < 2^52, so
    # u * 2^54 is an odd integer there: checks the 53-bit construction.
    u = oracle.uniforms(seed=1, particle=0, epoch=0, tag=0, n=20_000)
    small = u[u < 0.5]
    k = small * 2.0 ** 54
    assert np.all(k == np.floor(k)) and np.all(k.astype(np.int64) % 2 == 1)


def test_stream_layout_block_halves():
    # draw d comes from Philox block d>>1 with counter (b, t, n, tag), half d&1
    seed, n, t, tag = 0x1234_5678_9ABC, 17, 5, 0
    u = oracle.uniforms(seed, n, t, tag, 6)
    for d in range(6):
        blk = oracle.philox([d >> 1, t, n, tag], [seed & 0xFFFFFFFF, seed >> 32])
        x, y = (blk[0], blk[1]) if d % 2 == 0 else (blk[2], blk[3])
        z = int(x) ^ (int(y) << 21)
        assert z < 2 ** 53
        assert abs(u[d] - (z + 0.5) / 2.0 ** 53) <= 2.0 ** -53


def test_streams_distinct_per_particle_epoch_tag():
    a = oracle.uniforms(1, 0, 0, 0, 4)
    assert not np.array_equal(a, oracle.uniforms(1, 1, 0, 0, 4))
    assert not np.array_equal(a, oracle.uniforms(1, 0, 1, 0, 4))
    assert not np.array_equal(a, oracle.uniforms(1, 0, 0, 1, 4))
    assert not np.array_equal(a, oracle.uniforms(2, 0, 0, 0, 4))


def test_worked_values():
    # SURVEY §8(c.2b) worked values (computed there by a KAT-verified Philox)
    u = oracle.uniforms(0, 0, 0, 0, 2)
    assert u[0] == pytest.approx(0.88052026840093833, abs=1e-16)
    assert u[1] == pytest.approx(0.60548199590756147, abs=1e-16)
    assert oracle.uniforms(1, 0, 0, 1, 1)[0] == pytest.approx(0.11725545578469382, abs=1e-16)
