"""Pins for the 7th-order taper (N1).

The taper is the unique degree-7 polynomial with T(0)=1, T(R)=0 and vanishing
1st-3rd derivatives at both ends.  Its values at x = 1/4, 1/2,
3/4 follow from those 8 constraints; the test solves the constraints itself
in exact rationals (independent of the oracle's coefficients).
"""
import json
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle

R = 10.0
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _solve_taper_coeffs():
    # unknown a0..a7; rows: T(0)=1, T'(0)=T''(0)=T'''(0)=0, T(1)=0, T'(1)=T''(1)=T'''(1)=0
    rows, rhs = [], []
    for x, val in ((0, 1), (1, 0)):
        for d in range(4):
            row = []
            for k in range(8):
                if k < d:
                    row.append(Fr(0))
                else:
                    c = Fr(1)
                    for m in range(d):
                        c *= (k - m)
                    row.append(c * Fr(x) ** (k - d) if k - d > 0 else c)
            rows.append(row)
            rhs.append(Fr(val if d == 0 else 0))
    # Gauss-Jordan in exact arithmetic
    n = 8
    A = [r + [b] for r, b in zip(rows, rhs)]
    for c in range(n):
        p = next(r for r in range(c, n) if A[r][c] != 0)
        A[c], A[p] = A[p], A[c]
        A[c] = [v / A[c][c] for v in A[c]]
        for r in range(n):
            if r != c and A[r][c] != 0:
                A[r] = [a - A[r][c] * b for a, b in zip(A[r], A[c])]
    return [A[k][n] for k in range(n)]


COEF = _solve_taper_coeffs()


def _exact(x):
    return sum(c * Fr(x) ** k for k, c in enumerate(COEF))


@pytest.mark.parametrize("x", [Fr(0), Fr(1, 4), Fr(1, 2), Fr(3, 4), Fr(1), Fr(1, 8), Fr(7, 16)])
def test_taper_exact_rationals(x):
    t, _ = oracle.taper(float(x) * R, R)
    assert abs(t - float(_exact(x))) <= 4e-16


def test_taper_known_rationals():
    assert _exact(Fr(1, 2)) == Fr(1, 2)
    assert _exact(Fr(1, 4)) == Fr(3807, 4096)
    assert _exact(Fr(3, 4)) == Fr(289, 4096)


@pytest.mark.parametrize("case", GOLD["taper"])
def test_taper_golden(case):
    t, _ = oracle.taper(case["x"] * R, R)
    assert t == float(Fr(case["tap"]))


def test_taper_symmetry_and_monotone():
    xs = np.linspace(0, 1, 1001)
    t = np.array([oracle.taper(x * R, R)[0] for x in xs])
    # evaluation as written sums terms up to 210 in magnitude: rounding bound ~1e-13
    assert np.all(np.abs(t + t[::-1] - 1) < 1e-13)
    assert np.all(np.diff(t) <= 1e-16)


def test_taper_derivative_fd():
    h = 1e-4  # truncation ~h^2 T'''/6 ~ 2e-9; rounding ~1e-14/h
    for r in np.linspace(0.3, 9.7, 40):
        _, d = oracle.taper(r, R)
        fd = (oracle.taper(r + h, R)[0] - oracle.taper(r - h, R)[0]) / (2 * h)
        assert abs(d - fd) < 1e-8


def test_taper_flat_ends():
    # first three derivatives vanish at both ends: dTap ~ O(x^3) near 0 and O((1-x)^3) near 1
    for r in (0.0, R):
        assert oracle.taper(r, R)[1] == 0.0
    e = 1e-3
    assert abs(oracle.taper(e * R, R)[1]) < 1e-6 * 1.0
    assert abs(oracle.taper((1 - e) * R, R)[1]) < 1e-6 * 1.0
