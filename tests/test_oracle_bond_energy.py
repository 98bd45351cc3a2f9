"""Pins of the oracle's bond energy and its forces (O8, SURVEY.md §8(f) NEXT-1;
the bond part of "Aggregate Forces").

Pinned against things other than the oracle's own code:
  * central finite differences of the total bond energy (forces, at a fixed
    bond set) and of the per-bond energy in r, S_i, S_j (each partial);
  * special cases that reduce E1 to the linear form -sum(De_s BOs + De_p BOpi
    + De_pp BOpipi) over the corrected bond orders of the separately pinned
    B4-B8 path (orc_bo_correct): p_be1 = 0, and p_be2 -> 0 (BOs^p_be2 = 1);
  * Newton's third law, translation and relabelling invariance, zero forces
    at zero bond energies.
"""
import numpy as np
import pytest

import gen
import oracle

CUT = dict(r_nonb=6.0, r_bond=5.0, bo_cut=0.01)   # box 13 A > 2 r_nonb: ~215 atoms


@pytest.fixture(scope="module")
def small():
    return gen.make_system(215, (13.0, 13.0, 13.0), gen.SEED_BASE + 501)


@pytest.fixture(scope="module")
def params():
    return gen.make_params()


@pytest.fixture(scope="module")
def bparams():
    return gen.make_bond_params()


def _energy(sys_, params, bparams):
    E, F, ref = oracle.evaluate_bond_energy(sys_, params, bparams, CUT)
    return E, F, ref


def _bond_keys(ref):
    n = len(ref["brow"]) - 1
    rows = np.repeat(np.arange(n), np.diff(ref["brow"]))
    return set(zip(rows.tolist(), ref["bcol"].tolist()))


def test_forces_match_finite_differences(small, params, bparams):
    """Central differences with Richardson extrapolation (steps h and 2h; the
    steep B1 powers, p_bo6 up to 40, make the h^2 term visible)."""
    E0, F, ref0 = _energy(small, params, bparams)
    keys0 = _bond_keys(ref0)
    assert len(keys0) > 200
    h = 1e-5
    rng = np.random.default_rng(5)
    checked = 0
    for i in rng.choice(len(small.pos), 12, replace=False):
        for k in range(3):
            e = {}
            same = True
            for step in (h, -h, 2 * h, -2 * h):
                s = gen.System(small.pos.copy(), small.type, small.q, small.box)
                s.pos[i, k] += step
                Ek, _, refk = _energy(s, params, bparams)
                same &= _bond_keys(refk) == keys0
                e[step] = Ek
            if not same:   # the displacement moved a bond across bo_cut / r_bond: E jumps there (reading 2A)
                continue
            d1 = (e[h] - e[-h]) / (2 * h)
            d2 = (e[2 * h] - e[-2 * h]) / (4 * h)
            fd = -(4 * d1 - d2) / 3
            assert abs(fd - F[i, k]) <= 1e-6 * max(1.0, abs(F[i, k])), (i, k, fd, F[i, k])
            checked += 1
    assert checked >= 30


def _canon(ref, type_):
    n = len(ref["brow"]) - 1
    for i in range(n):
        for e in range(ref["brow"][i], ref["brow"][i + 1]):
            j = ref["bcol"][e]
            if j > i:
                yield i, j, e


@pytest.mark.parametrize("which", ["r", "Si", "Sj"])
def test_pair_partials_match_finite_differences(small, params, bparams, which):
    """de/dr at fixed S, de/dS_i, de/dS_j of single bonds, by central differences."""
    _, _, ref = _energy(small, params, bparams)
    dl = ref["delta"]
    pos, box = ref["pos"], small.box
    rng = np.random.default_rng(11)
    bonds = list(_canon(ref, small.type))
    for idx in rng.choice(len(bonds), 25, replace=False):
        i, j, e = bonds[idx]
        d = np.array([oracle.min_image(pos[j, k] - pos[i, k], box[k]) for k in range(3)])
        r = float(np.sqrt(d @ d))
        ti, tj = small.type[i], small.type[j]
        args = [dl[i, 0], dl[i, 1], dl[j, 0], dl[j, 1]]
        out = oracle.bond_energy_pair(r, ref["raw"][e], *args, ti, tj, params, bparams)
        h = 1e-6
        if which == "r":
            ep = oracle.bond_energy_pair(r + h, oracle.bo_raw(r + h, ti, tj, params), *args, ti, tj, params, bparams)[0]
            em = oracle.bond_energy_pair(r - h, oracle.bo_raw(r - h, ti, tj, params), *args, ti, tj, params, bparams)[0]
            exact = out[1]
        else:
            sh = np.array([h, h, 0, 0]) if which == "Si" else np.array([0, 0, h, h])
            ap, am = list(np.array(args) + sh), list(np.array(args) - sh)
            ep = oracle.bond_energy_pair(r, ref["raw"][e], *ap, ti, tj, params, bparams)[0]
            em = oracle.bond_energy_pair(r, ref["raw"][e], *am, ti, tj, params, bparams)[0]
            exact = out[2] if which == "Si" else out[3]
        fd = (ep - em) / (2 * h)
        assert abs(fd - exact) <= 1e-6 * max(1.0, abs(exact)), (which, i, j, fd, exact)


def test_dbo_dr_matches_finite_differences(params):
    for (ti, tj) in [(0, 0), (0, 3), (1, 2), (3, 3)]:
        for r in (0.9, 1.2, 1.6, 2.1):
            raw = oracle.bo_raw(r, ti, tj, params)
            out = oracle.bond_energy_pair(r, raw, 0.1, 0.1, -0.2, -0.2, ti, tj, params, gen.make_bond_params())
            h = 1e-6
            fd = (oracle.bo_raw(r + h, ti, tj, params)[3] - oracle.bo_raw(r - h, ti, tj, params)[3]) / (2 * h)
            assert abs(fd - out[4]) <= 1e-7 * max(1.0, abs(out[4]))


def _linear_energy(ref, params, bp, type_):
    """-sum (De_s BOs + De_p BOpi + De_pp BOpipi) from the pinned corrected bond orders."""
    corr = ref["corr"]   # [B][4] = BO, BOs, BOpi, BOpipi
    E = 0.0
    for i, j, e in _canon(ref, type_):
        ti, tj = type_[i], type_[j]
        E -= params.De[ti, tj] * corr[e, 1] + bp.De_pi[ti, tj] * corr[e, 2] + bp.De_pipi[ti, tj] * corr[e, 3]
    return E


@pytest.mark.parametrize("case", ["p_be1=0", "p_be2->0"])
def test_reduces_to_linear_form(small, params, bparams, case):
    bp = bparams.copy()
    if case == "p_be1=0":
        bp.p_be1[:] = 0.0
    else:
        bp.p_be2[:] = 1e-300   # BOs^p_be2 = 1 for every BOs > 0: exp(p_be1 (1 - 1)) = 1
    E, _, ref = _energy(small, params, bp)
    if case == "p_be2->0":
        assert np.all(ref["corr"][:, 1] > 0)
    El = _linear_energy(ref, params, bp, small.type)
    assert abs(E - El) <= 1e-12 * abs(El)


def test_newton_translation_relabel(small, params, bparams):
    E, F, _ = _energy(small, params, bparams)
    assert np.all(np.abs(F.sum(0)) <= 1e-11 * np.abs(F).sum())
    s = gen.System(small.pos + np.array([3.1, -7.7, 11.9]), small.type, small.q, small.box)
    E2, F2, _ = _energy(s, params, bparams)
    assert abs(E2 - E) <= 1e-10 * abs(E)
    assert np.all(np.abs(F2 - F) <= 1e-8 * (1 + np.abs(F)))
    perm = np.random.default_rng(3).permutation(len(small.pos))
    s = gen.System(small.pos[perm].copy(), small.type[perm].copy(), small.q[perm].copy(), small.box)
    E3, F3, _ = _energy(s, params, bparams)
    assert abs(E3 - E) <= 1e-10 * abs(E)
    assert np.all(np.abs(F3 - F[perm]) <= 1e-8 * (1 + np.abs(F[perm])))


def test_zero_bond_energies_give_zero(small, params, bparams):
    p = params.copy()
    p.De[:] = 0.0
    bp = bparams.copy()
    bp.De_pi[:] = 0.0
    bp.De_pipi[:] = 0.0
    E, F, _ = _energy(small, p, bp)
    assert E == 0.0 and np.all(F == 0.0)


@pytest.mark.parametrize("m", [2.0, 3.0, 0.5])
def test_e1_closed_form_sign_of_p_be1(params, bparams, m):
    """E1 at BOs = m^(1/p_be2): BOs^p_be2 = m, so e = -De_s BOs exp(p_be1 (1 - m))
    - De_p BOpi - De_pp BOpipi.  Delta' = 0 gives f1 = 1 exactly and
    Delta'boc = -1000 gives f4 = f5 = 1 exactly (exp(< -700) = 0), so the
    corrected orders are the raw terms: BOs = raw sigma, BOpi, BOpipi.  At
    m = 2 the factor is exp(-p_be1): a flipped sign of p_be1 (exp(+p_be1)) or a
    misplaced p_be2 fails."""
    for ti, tj in [(0, 0), (0, 2), (1, 3)]:
        b1, b2 = bparams.p_be1[ti, tj], bparams.p_be2[ti, tj]
        assert abs(b1) > 1e-3
        bs = m ** (1.0 / b2)
        bpi, bpp = 0.25, 0.125
        raw = np.array([bs, bpi, bpp, (bs + bpi) + bpp])
        out = oracle.bond_energy_pair(1.3, raw, 0.0, -1000.0, 0.0, -1000.0, ti, tj, params, bparams)
        # BOs = BO - BOpi - BOpipi reconstructs raw sigma to rounding
        want = -params.De[ti, tj] * bs * np.exp(b1 * (1.0 - m)) - bparams.De_pi[ti, tj] * bpi \
            - bparams.De_pipi[ti, tj] * bpp
        assert abs(out[0] - want) <= 1e-13 * abs(want), (ti, tj, out[0], want)
        # and the sigma factor alone at m = 2 is exp(-p_be1), not exp(+p_be1)
        if m == 2.0:
            sig = (out[0] + bparams.De_pi[ti, tj] * bpi + bparams.De_pipi[ti, tj] * bpp) / (-params.De[ti, tj] * bs)
            assert abs(sig - np.exp(-b1)) <= 1e-12 * np.exp(-b1)
            assert abs(sig - np.exp(b1)) > 1e-6
