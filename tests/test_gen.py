"""Seeded input generator (gen/): determinism, recipe properties.  Not the method."""
import numpy as np
import pytest

import gen


def test_splitmix64_reference_vector():
    # SplitMix64 (Steele/Lea/Flood; Vigna's splitmix64.c) from state 0 yields
    # 0xE220A8397B1DCDAF first; u = (z >> 11) * 2^-53.
    u = gen.uniforms(0, 1)[0]
    assert u == (0xE220A8397B1DCDAF >> 11) * 2.0 ** -53


def test_uniforms_range_and_determinism():
    a = gen.uniforms(123, 10000)
    assert a.min() >= 0.0 and a.max() < 1.0
    assert np.array_equal(a, gen.uniforms(123, 10000))
    assert abs(a.mean() - 0.5) < 0.01


def test_config0_recipe(c0):
    n = 2088
    assert c0.pos.shape == (n, 3)
    assert np.all(c0.pos >= 0) and np.all(c0.pos < c0.box)
    # C5H8N4O12 composition, 72 formula units
    counts = np.bincount(c0.type, minlength=4)
    assert counts.tolist() == [72 * 5, 72 * 8, 72 * 4, 72 * 12]
    assert abs(c0.q.sum()) < 1e-12
    assert c0.q.min() >= -0.53 and c0.q.max() <= 0.53
    # minimum separation 0.9 A (brute force, minimum image)
    d = c0.pos[:, None, :] - c0.pos[None, :, :]
    d -= c0.box * np.round(d / c0.box)
    r2 = (d ** 2).sum(-1) + np.eye(n) * 1e9
    assert r2.min() >= 0.81


def test_determinism():
    a = gen.make_system(500, (21.0, 22.0, 23.0), 7)
    b = gen.make_system(500, (21.0, 22.0, 23.0), 7)
    assert np.array_equal(a.pos, b.pos) and np.array_equal(a.q, b.q)
    c = gen.make_system(500, (21.0, 22.0, 23.0), 8)
    assert not np.array_equal(a.pos, c.pos)


def test_params_ranges(params):
    p = params
    assert p.ntypes == 4
    for f, lo, hi in [("r_sigma", 0.9, 1.5), ("r_pi", 1.1, 1.3), ("r_pipi", 1.0, 1.2), ("gamma", 0.5, 1.0),
                      ("r_vdw", 1.5, 2.1), ("eps", 0.05, 0.2), ("alpha", 9, 12), ("gamma_w", 1.5, 8),
                      ("b131", 2, 10), ("b132", 1, 10), ("b133", 0.5, 10)]:
        a = getattr(p, f)
        assert np.all(a >= lo) and np.all(a <= hi), f
    for f, lo, hi in [("p_bo1", -0.15, -0.05), ("p_bo2", 5, 9), ("p_bo3", -0.35, -0.10), ("p_bo4", 5, 12),
                      ("p_bo5", -0.45, -0.20), ("p_bo6", 10, 40), ("De", 50, 150)]:
        a = getattr(p, f)
        assert np.all(a >= lo) and np.all(a <= hi), f
        assert np.array_equal(a, a.T), f
    assert p.val.tolist() == [4.0, 1.0, 3.0, 2.0]


@pytest.mark.parametrize("k", [1, 2])
def test_configs_density(k):
    s = gen.make_config(k)
    rho = len(s.pos) / np.prod(s.box)
    assert abs(rho - 0.0978) < 0.0015
