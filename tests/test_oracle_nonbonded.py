"""Pins for oracle O6 (Alg. 1 / Alg. 2 nonbonded energies and forces).

Independent pins: central finite differences of the total energy (small
systems, charges frozen), Newton's third law,
translation / relabelling / mirror invariance, the half-list
scatter (Alg. 2) against a per-atom full-neighbourhood gather, and exact
charge scaling.
"""
import numpy as np
import pytest

import gen
import oracle

CUT = gen.CUTOFFS


def _energy(s, params):
    return oracle.evaluate(s, params, CUT)["E"].sum()


@pytest.mark.parametrize("seed,n", [(1, 8), (2, 24), (3, 64)])
def test_forces_finite_difference(params, seed, n):
    s = gen.make_system(n, (20.5, 21.0, 21.5), 500 + seed)
    F = oracle.evaluate(s, params, CUT)["F"]
    h = 1e-5
    rng = np.random.default_rng(seed)
    for a in rng.choice(n, size=min(n, 6), replace=False):
        for k in range(3):
            sp = gen.System(s.pos.copy(), s.type, s.q, s.box)
            sm = gen.System(s.pos.copy(), s.type, s.q, s.box)
            sp.pos[a, k] += h
            sm.pos[a, k] -= h
            fd = -(_energy(sp, params) - _energy(sm, params)) / (2 * h)
            assert abs(F[a, k] - fd) <= 1e-6 * max(1.0, abs(F[a, k])), (a, k, F[a, k], fd)


def test_newton_third_law(c0_oracle):
    F = c0_oracle["F"]
    assert np.all(np.abs(F.sum(0)) <= 1e-12 * np.abs(F).sum())


def test_translation_invariance(c0, params, c0_oracle):
    shift = np.array([3.7, 11.2, 25.9])
    s2 = gen.System(oracle.wrap(c0.pos + shift, c0.box), c0.type, c0.q, c0.box)
    o2 = oracle.evaluate(s2, params, CUT)
    E1, E2 = c0_oracle["E"], o2["E"]
    assert np.all(np.abs(E2 - E1) <= 1e-12 * np.abs(E1))
    F1, F2 = c0_oracle["F"], o2["F"]
    assert np.all(np.abs(F2 - F1) <= 1e-9 * (1 + np.abs(F1)))
    assert len(o2["hcol"]) == len(c0_oracle["hcol"])


def test_relabel_invariance(c0, params, c0_oracle):
    perm = np.random.default_rng(0).permutation(len(c0.pos))
    s2 = gen.System(c0.pos[perm], c0.type[perm], c0.q[perm], c0.box)
    o2 = oracle.evaluate(s2, params, CUT)
    assert np.all(np.abs(o2["E"] - c0_oracle["E"]) <= 1e-12 * np.abs(c0_oracle["E"]))
    assert np.all(np.abs(o2["F"] - c0_oracle["F"][perm]) <= 1e-9 * (1 + np.abs(c0_oracle["F"][perm])))
    # bonds: same multiset of corrected BO
    a = np.sort(o2["corr"][:, 0])
    b = np.sort(c0_oracle["corr"][:, 0])
    assert np.all(np.abs(a - b) <= 1e-13)


def test_mirror_invariance(params):
    s = gen.make_system(400, (21.0, 21.0, 21.0), 77)
    o = oracle.evaluate(s, params, CUT)
    pos2 = s.pos.copy()
    pos2[:, 0] = s.box[0] - pos2[:, 0]
    s2 = gen.System(oracle.wrap(pos2, s.box), s.type, s.q, s.box)
    o2 = oracle.evaluate(s2, params, CUT)
    assert np.all(np.abs(o2["E"] - o["E"]) <= 1e-12 * np.abs(o["E"]))
    F2 = o2["F"].copy()
    F2[:, 0] *= -1
    assert np.all(np.abs(F2 - o["F"]) <= 1e-9 * (1 + np.abs(o["F"])))


def test_scatter_equals_gather(c0, params, c0_oracle):
    pos = c0_oracle["pos"]
    tot = np.zeros(2)
    for i in range(len(pos)):
        F, Eh = oracle.atom_force(i, pos, c0.type, c0.q, c0.box, params, 10.0)
        tot += Eh
        if i % 97 == 0:
            assert np.all(np.abs(F - c0_oracle["F"][i]) <= 1e-10 * (1 + np.abs(F)))
    assert np.all(np.abs(tot - c0_oracle["E"]) <= 1e-11 * np.abs(c0_oracle["E"]))


def test_charge_scaling_bitwise(c0, params, c0_oracle):
    o = c0_oracle
    E2, _ = oracle.nonbonded(o["pos"], c0.type, 2 * c0.q, c0.box, params, 10.0, o["hrow"], o["hcol"])
    assert E2[1] == 4 * o["E"][1] and E2[0] == o["E"][0]
    E0, F0 = oracle.nonbonded(o["pos"], c0.type, 0 * c0.q, c0.box, params, 10.0, o["hrow"], o["hcol"])
    assert E0[1] == 0.0


def test_isolated_pair_matches_pair_function(params):
    L = 30.0
    pos = np.array([[1.0, 2.0, 3.0], [1.0 + 3.0, 2.0 + 4.0, 3.0]])  # r = 5 exactly
    typ = np.array([1, 3], np.int32)
    q = np.array([0.25, -0.5])
    s = gen.System(pos, typ, q, np.array([L, L, L]))
    o = oracle.evaluate(s, params, CUT)
    e, d = oracle.pair(5.0, 1, 3, 0.25, -0.5, params, 10.0)
    assert np.array_equal(o["E"], e)
    g = d / 5.0
    assert np.array_equal(o["F"][0], g * np.array([3.0, 4.0, 0.0]))
    assert np.array_equal(o["F"][1], -g * np.array([3.0, 4.0, 0.0]))
