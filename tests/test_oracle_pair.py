"""Pins for the pair terms N2-N5 (shielded vdW, shielded Coulomb, tapered pair).

Independent pins: the vdW minimum (u = 0 gives e_v = -D and de_v/dr = 0),
the unshielded limits that reduce to the textbook Morse and Coulomb forms,
central finite differences of E(r), exact charge scaling.
"""
import numpy as np
import pytest

import gen
import oracle

R = 10.0


def _pair_consts(p, ti, tj):
    D = np.sqrt(p.eps[ti] * p.eps[tj])
    alpha = np.sqrt(p.alpha[ti] * p.alpha[tj])
    rvdw = 2 * np.sqrt(p.r_vdw[ti] * p.r_vdw[tj])
    gw = np.sqrt(p.gamma_w[ti] * p.gamma_w[tj])
    return D, alpha, rvdw, gw


@pytest.mark.parametrize("ti,tj", [(0, 0), (0, 1), (1, 3), (2, 3), (3, 3)])
def test_vdw_minimum_is_minus_D(params, ti, tj):
    D, alpha, rvdw, gw = _pair_consts(params, ti, tj)
    p = params.p_vdw1
    rstar = (rvdw ** p - gw ** (-p)) ** (1 / p)
    ev, dev = oracle.vdw(rstar, ti, tj, params)
    assert abs(ev + D) < 1e-13 * D
    assert abs(dev) < 1e-12 * D * alpha
    # it is the minimum: neighbours are higher
    assert oracle.vdw(rstar * 1.01, ti, tj, params)[0] > ev
    assert oracle.vdw(rstar * 0.99, ti, tj, params)[0] > ev
    # tapered pair: E_v = -D Tap(r*), dE_v/dr = -D dTap(r*)  (q = 0 removes Coulomb)
    e, dEdr = oracle.pair(rstar, ti, tj, 0.0, 0.0, params, R)
    tap, dtap = oracle.taper(rstar, R)
    assert abs(e[0] + D * tap) < 1e-13 * D and e[1] == 0.0
    assert abs(dEdr + D * dtap) < 1e-12 * D * alpha


def test_vdw_unshielded_is_morse(params):
    # gamma_w -> infinity: f13 -> r, e_v -> Morse D(e^{-2a(r-re)} - 2 e^{-a(r-re)}),
    # re = r_vdW, a = alpha / (2 r_vdW)
    p = params.copy()
    p.gamma_w = np.full(p.ntypes, 1e12)
    for ti, tj in [(0, 2), (1, 1)]:
        D, alpha, rvdw, _ = _pair_consts(p, ti, tj)
        a = alpha / (2 * rvdw)
        for r in (1.0, 2.5, rvdw, 5.0, 9.0):
            morse = D * (np.exp(-2 * a * (r - rvdw)) - 2 * np.exp(-a * (r - rvdw)))
            dmorse = D * (-2 * a * np.exp(-2 * a * (r - rvdw)) + 2 * a * np.exp(-a * (r - rvdw)))
            ev, dev = oracle.vdw(r, ti, tj, p)
            assert abs(ev - morse) < 1e-12 * max(1, abs(morse))
            assert abs(dev - dmorse) < 1e-11 * max(1, abs(dmorse))


def test_coulomb_unshielded_is_coulomb(params):
    p = params.copy()
    p.gamma = np.full(p.ntypes, 1e7)
    for r in (0.9, 1.7, 4.0, 9.5):
        k, dk = oracle.coulomb_kernel(r, 0, 3, p)
        assert abs(k - 1 / r) < 1e-14 / r
        assert abs(dk + 1 / r ** 2) < 1e-13 / r ** 2


def test_coulomb_shielding_bounded(params):
    # S^(-1/3) <= gamma_ij and -> gamma_ij as r -> 0 (shielded 1/r never diverges)
    g = np.sqrt(params.gamma[1] * params.gamma[2])
    k0, _ = oracle.coulomb_kernel(1e-8, 1, 2, params)
    assert abs(k0 - g) < 1e-12
    for r in np.linspace(0.5, 10, 20):
        assert oracle.coulomb_kernel(r, 1, 2, params)[0] < min(g, 1 / r) + 1e-15


def test_pair_fd(params):
    rng = np.random.default_rng(5)
    h = 1e-6
    for _ in range(200):
        ti, tj = rng.integers(0, 4, 2)
        qi, qj = rng.uniform(-0.5, 0.5, 2)
        r = rng.uniform(0.9, 9.99)
        e, d = oracle.pair(r, ti, tj, qi, qj, params, R)
        ep, _ = oracle.pair(r + h, ti, tj, qi, qj, params, R)
        em, _ = oracle.pair(r - h, ti, tj, qi, qj, params, R)
        fd = (ep.sum() - em.sum()) / (2 * h)
        assert abs(d - fd) <= 1e-6 * max(1.0, abs(d))


def test_pair_zero_at_cutoff(params):
    e, d = oracle.pair(R, 0, 1, 0.3, -0.2, params, R)
    assert e[0] == 0.0 and e[1] == 0.0 and d == 0.0


def test_charge_scaling_exact(params):
    for r in (1.1, 3.3, 7.7):
        e1, _ = oracle.pair(r, 2, 3, 0.3, -0.2, params, R)
        e2, _ = oracle.pair(r, 2, 3, 0.6, -0.4, params, R)
        assert e2[1] == 4 * e1[1] and e2[0] == e1[0]
        e0, _ = oracle.pair(r, 2, 3, 0.0, -0.2, params, R)
        assert e0[1] == 0.0


def test_pair_symmetric(params):
    for r in (1.3, 4.2):
        a, da = oracle.pair(r, 0, 3, 0.1, -0.3, params, R)
        b, db = oracle.pair(r, 3, 0, -0.3, 0.1, params, R)
        assert np.array_equal(a, b) and da == db
